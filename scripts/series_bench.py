"""Timing of the n-term series (ps_solve_series) on a BASELINE config.

For each nrhs: the two-term ps_solve (single dataflow program), ps_solve_series at n = 2 and
n = n_hi terms (per-operator launch sets), CUDA events on the solve stream after warm-up. The
cost of one extra term is (t(n_hi) - t(2)) / (n_hi - 2); its algorithmic work is one U
application, 16 (2 n_R + n_D + n_F) operator bytes + vector passes and 8 nrhs (2 n_R + n_D +
2 n_F) flop (include/ps.h ps_series_report), against the measured HBM / FP64 peaks.

  python scripts/series_bench.py --config C4 --nrhs 1 360 --terms 6
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
    ap.add_argument("--nrhs", type=int, nargs="+", default=[1, 360])
    ap.add_argument("--terms", type=int, default=6)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    import torch
    from hmgen.build import load_or_generate, read_rhs
    from paper_2109_04129_b200 import PsHandle
    warnings.simplefilter("ignore")
    meta = load_or_generate(a.config)
    B, _ = read_rhs(meta["rhs"])
    h = PsHandle(meta["hm"], device=0)
    h.setup()
    info = h.info()
    N = int(info["N"])
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm = float(peaks.get("hbm_gbs", 6548.2))
    except Exception:
        hbm = 6548.2
    fp64 = 37.02
    st = torch.cuda.Stream()
    out = []
    for R in a.nrhs:
        cols = np.arange(R) % B.shape[1]
        Bd = torch.from_numpy(np.ascontiguousarray(B[:, cols].T)).cuda().T
        Xd = torch.empty_like(Bd)

        def timed(fn):
            for _ in range(a.warmup):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                e0.record(st)
                for _ in range(a.steps):
                    fn()
                e1.record(st)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / a.steps

        t_prog = timed(lambda: h.solve(Bd, Xd, stream=st, want_norms=False))
        t2 = timed(lambda: h.solve_series(Bd, Xd, max_terms=2, stream=st))
        tn = timed(lambda: h.solve_series(Bd, Xd, max_terms=a.terms, stream=st))
        _, rep = h.solve_series(Bd, Xd, max_terms=a.terms, stream=st)
        t_term = (tn - t2) / (a.terms - 2)
        nR, nD, nF = info["nR"], info["nD"], info["nF"]
        by = 16.0 * (2 * nR + nD + nF) + 16.0 * 6 * N * R
        fl = 8.0 * R * (2 * nR + nD + 2 * nF)
        r = {"config": a.config, "N": N, "nrhs": R, "terms": a.terms,
             "ms_two_term_program": t_prog, "ms_series_2": t2, f"ms_series_{a.terms}": tn,
             "ms_per_extra_term": t_term, "launches_series": rep["launches"],
             "per_term": {"bytes": by, "flop": fl,
                          "hbm_frac": by / (t_term * 1e-3) / 1e9 / hbm,
                          "fp64_frac": fl / (t_term * 1e-3) / 1e12 / fp64},
             "N_nrhs_terms_per_s": N * R * a.terms / (tn * 1e-3),
             "it_norm_ratio_last": (rep["it_norm"][-1] / rep["it_norm"][-2]).tolist()[:4]}
        print(json.dumps(r), flush=True)
        out.append(r)
    h.close()


if __name__ == "__main__":
    main()
