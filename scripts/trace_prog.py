"""Per-work-item trace of the single-launch solve program (class 6):
  python scripts/trace_prog.py --config C2 [--nrhs 181] --out gpurun_out/trace_prog.npz"""
import argparse
import os
import sys
import warnings

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--nrhs", type=int, default=0)
    ap.add_argument("--out", default="gpurun_out/trace_prog.npz")
    args = ap.parse_args()
    warnings.simplefilter("ignore")
    import torch
    from hmgen.build import load_or_generate, read_rhs
    from paper_2109_04129_b200 import PsHandle
    meta = load_or_generate(args.config)
    B, _ = read_rhs(meta["rhs"])
    if args.nrhs:
        B = B[:, :args.nrhs]
    h = PsHandle(meta["hm"])
    h.setup()
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().T
    Xd = torch.empty_like(Bd)
    for _ in range(3):
        h.solve(Bd, Xd)
    h.profile(True)
    h.trace(6)
    h.solve(Bd, Xd)
    tr = h.trace_read()
    h.trace(-1)
    print("items", len(tr), h.profile_read()["solve_program"])
    np.savez(args.out, prog=tr)


if __name__ == "__main__":
    main()
