"""Timing of the RCS post-processing (ps_farfield) on a BASELINE config:
the monostatic sweep (direction c paired with column c) on the currents ps_solve returns, and
a bistatic cut (--bistatic directions for every column), CUDA events after warm-up.
Work per (direction, sample, column): one FP64 sincos (direction-sample pair) + 13 FMA
(phase 3, complex current x phase 4, 3 complex accumulations 6): reported as sample-pairs/s
and as the FMA rate against the measured FP64 peak (an ALU-bound kernel; the sincos is extra).

  python scripts/rcs_bench.py --config C4 --bistatic 181
"""
import argparse
import json
import os
import sys
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--bistatic", type=int, default=181)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    import torch
    from hmgen.build import CONFIGS, load_or_generate, make_mesh, plane_wave_dirs, read_rhs, rwg_basis
    from paper_2109_04129_b200 import PsHandle, farfield
    warnings.simplefilter("ignore")
    cfg = CONFIGS[a.config]
    meta = load_or_generate(a.config)
    B, _ = read_rhs(meta["rhs"])
    h = PsHandle(meta["hm"], device=0)
    h.setup()
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().T
    Xd = torch.empty_like(Bd)
    h.solve(Bd, Xd)
    h.close()
    m = make_mesh(cfg)
    bs = rwg_basis(m)
    _, khat, _ = plane_wave_dirs(cfg)
    g = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (m.nodes, m.tris, bs.tp, bs.tm, bs.vp, bs.vm)]
    eta = 120 * np.pi
    N, R = bs.N, B.shape[1]

    def timed(fn):
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.steps

    rh_m = torch.from_numpy(-np.asarray(khat)).cuda()
    ms_m = timed(lambda: farfield(*g, cfg.k, eta, Xd, rh_m, mono=True))
    th = np.deg2rad(np.linspace(0, 180, a.bistatic))
    rh_b = torch.from_numpy(np.stack([np.sin(th), 0 * th, np.cos(th)], 1)).cuda()
    ms_b = timed(lambda: farfield(*g, cfg.k, eta, Xd, rh_b, mono=False))
    fp64 = 37.02
    out = {"config": a.config, "N": N, "samples": 14 * N,
           "monostatic": {"directions": R, "ms": ms_m, "pairs_per_s": R * 14 * N / (ms_m * 1e-3),
                          "fma_tflops": 26 * R * 14 * N / (ms_m * 1e-3) / 1e12,
                          "fma_frac_fp64": 26 * R * 14 * N / (ms_m * 1e-3) / 1e12 / fp64},
           "bistatic": {"directions": a.bistatic, "columns": R, "ms": ms_b,
                        "pairs_per_s": a.bistatic * 14 * N / (ms_b * 1e-3),
                        "fma_tflops": (6 + 20 * R) * a.bistatic * 14 * N / (ms_b * 1e-3) / 1e12,
                        "fma_frac_fp64": (6 + 20 * R) * a.bistatic * 14 * N / (ms_b * 1e-3) / 1e12 / fp64},
           "note": "ALU-bound; flop = 2 x FMA count (phase 3 FMA per direction-sample, 10 per column), "
                   "sincos not counted; FP64 peak 37.02 TF (profiles/r1/fp64_peak_b200.json)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
