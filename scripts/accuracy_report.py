"""Truncation size of the two-term series (SURVEY §8(c) "truncation size: reported number";
the paper's §V.A metric ||SOL_dir - SOL_ps|| / ||SOL_dir||).

For each config: the oracle's two-term solution x2 (oracle.solve, Eqs. 24-36) against the
dense-LU solution of the full H-matrix system Z = Z_N + Z_F (oracle.dense; LAPACK), per RHS
column, with the ratio ||it_1|| / ||it_0|| of Eq. 45 next to it. Calls only oracle/ (and the
shared input generator); writes tests/golden/accuracy.json.

  python scripts/accuracy_report.py C1 C2
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def report(name):
    from hmgen.build import load_or_generate, read_rhs
    from oracle import compute_scaling, read_hm, solve
    from oracle.dense import dense_ZF, dense_ZN, direct_solve
    meta = load_or_generate(name)
    H = read_hm(meta["hm"])
    B, ang = read_rhs(meta["rhs"])
    t0 = time.time()
    res = solve(H, compute_scaling(H), B)
    Z = dense_ZN(H)
    Z += dense_ZF(H)
    xd = direct_solve(Z, B)
    del Z
    err = np.linalg.norm(res.x - xd, axis=0) / np.linalg.norm(xd, axis=0)
    return {"config": name, "N": int(H.N), "nrhs": int(B.shape[1]),
            "rel_err_two_term_vs_dense_LU": {"min": float(err.min()), "median": float(np.median(err)),
                                            "max": float(err.max())},
            "ratio_it1_it0": {"min": float(res.ratio.min()), "median": float(np.median(res.ratio)),
                              "max": float(res.ratio.max())},
            "per_column": [{"theta_phi_deg": [float(a) for a in ang[c]], "rel_err": float(err[c]),
                            "ratio": float(res.ratio[c])} for c in range(B.shape[1])],
            "seconds": time.time() - t0}


if __name__ == "__main__":
    out = os.path.join(ROOT, "tests", "golden", "accuracy.json")
    d = {}
    if os.path.exists(out):
        with open(out) as f:
            d = json.load(f)
    d["_what"] = ("two-term power series (oracle) vs dense LU of Z = Z_N + Z_F: ||x2 - Z^-1 b|| / ||Z^-1 b|| per "
                  "plane-wave column (PAPER.md:313 metric); written by scripts/accuracy_report.py (oracle only)")
    for name in sys.argv[1:] or ["C1", "C2"]:
        d[name] = report(name)
        print(name, json.dumps({k: d[name][k] for k in ("N", "nrhs", "rel_err_two_term_vs_dense_LU",
                                                         "ratio_it1_it0")}), flush=True)
    with open(out, "w") as f:
        json.dump(d, f, indent=1)
