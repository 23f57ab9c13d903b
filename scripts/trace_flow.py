"""Record per-work-item timestamps of the persistent dataflow kernel (debug).

  python scripts/trace_flow.py [--config C2] [--nrhs 181] [--out gpurun_out/trace_C2.npz]
"""
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
    ap.add_argument("--out", default="")
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
    out = {}
    names = ["fwd", "bwd", "dinv", "far1", "far2"]
    for c, nm in enumerate(names):
        h.profile(True)
        h.trace(c)
        h.solve(Bd, Xd)
        out[nm] = h.trace_read()
        h.trace(-1)
        prof = h.profile_read()
        h.profile(False)
        tr = out[nm]
        span = (tr[:, 5].max() - tr[:, 2].min()) / 1e3 if len(tr) else 0
        print(f"{nm}: items={len(tr)} span={span:.1f} us  prof={prof}")
    path = args.out or f"gpurun_out/trace_{args.config}.npz"
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez(path, **out)
    print("saved", path)


if __name__ == "__main__":
    main()
