"""Small C1 workload for compute-sanitizer (memcheck / racecheck / synccheck):
setup + solves at nrhs = 1 (narrow warp-specialised kernel), 40 (wide DFMA/DMMA
kernel) and the per-operator stage tables (ps_apply), each compared with the oracle.

  compute-sanitizer --tool memcheck python scripts/sanitize_c1.py
"""
import os
import sys
import warnings

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    warnings.simplefilter("ignore")
    import torch
    from hmgen.build import load_or_generate
    from hmgen.synth import random_rhs
    from oracle import compute_scaling, read_hm, solve
    from paper_2109_04129_b200 import PS_OP_U, PsHandle
    meta = load_or_generate("C1")
    H = read_hm(meta["hm"])
    S = compute_scaling(H)
    h = PsHandle(meta["hm"])
    h.setup()
    worst = 0.0
    for nrhs in (1, 40):
        B = random_rhs(H.N, nrhs, 3)
        Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().T
        Xd = torch.empty_like(Bd)
        h.solve(Bd, Xd)
        x = Xd.T.cpu().numpy().T
        ref = solve(H, S, B)
        err = np.linalg.norm(x - ref.x, axis=0) / np.linalg.norm(ref.x, axis=0)
        worst = max(worst, float(err.max()))
        Yd = torch.empty_like(Bd)
        h.apply(PS_OP_U, Bd, Yd)
    h.close()
    print(f"sanitize_c1: max rel L2 vs oracle {worst:.3e}")
    assert worst <= 1e-11


if __name__ == "__main__":
    main()
