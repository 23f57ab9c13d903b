"""One ps_solve inside a cudaProfilerStart/Stop range, for ncu captures:

  ncu --profile-from-start off --set full -k regex:flow_kernel -o gpurun_out/x \
      python scripts/ncu_solve.py --config C2 [--nrhs 181]

Setup and warm-up solves run outside the profiled range.
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
    ap.add_argument("--solves", type=int, default=1)
    args = ap.parse_args()
    warnings.simplefilter("ignore")
    import torch
    from hmgen.build import load_or_generate, read_rhs
    from paper_2109_04129_b200 import PsHandle
    meta = load_or_generate(args.config)
    B, _ = read_rhs(meta["rhs"])
    if args.nrhs:
        B = np.tile(B, (1, (args.nrhs + B.shape[1] - 1) // B.shape[1]))[:, :args.nrhs]
    h = PsHandle(meta["hm"])
    h.setup()
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().T
    Xd = torch.empty_like(Bd)
    for _ in range(2):
        h.solve(Bd, Xd)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(args.solves):
        h.solve(Bd, Xd)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    h.close()
    print("ok", args.config, B.shape)


if __name__ == "__main__":
    main()
