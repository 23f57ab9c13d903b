"""Per-operator device time and achieved rate of the stage-table solve (PS_SOLVE=stages:
one launch per operator class, CUDA events per launch via ps_profile), next to the
single-launch program time of the default path.

  python scripts/class_times.py --config C4 [--nrhs 360]
"""
import argparse
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(args):
    import warnings
    warnings.simplefilter("ignore")
    import numpy as np
    import torch
    from hmgen.build import load_or_generate, read_rhs
    from paper_2109_04129_b200 import PsHandle
    meta = load_or_generate(args.config)
    B, _ = read_rhs(meta["rhs"])
    if args.nrhs:
        B = np.tile(B, (1, -(-args.nrhs // B.shape[1])))[:, :args.nrhs]
    h = PsHandle(meta["hm"])
    h.setup()
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().T
    Xd = torch.empty_like(Bd)
    for _ in range(3):
        h.solve(Bd, Xd)
    h.profile(True)
    for _ in range(args.reps):
        h.solve(Bd, Xd)
    p = h.profile_read()
    out = {}
    for c, v in p.items():
        if v["launches"]:
            ms = v["ms"] / args.reps
            out[c] = {"ms": ms, "launches": v["launches"] / args.reps, "gflop": v["flops"] / args.reps / 1e9,
                      "tflops": v["flops"] / args.reps / (ms * 1e-3) / 1e12 if ms > 0 else 0,
                      "op_GB": v["bytes"] / args.reps / 1e9,
                      "GBs": v["bytes"] / args.reps / (ms * 1e-3) / 1e9 if ms > 0 else 0}
    print(json.dumps({"config": args.config, "nrhs": B.shape[1], "mode": os.environ.get("PS_SOLVE", "program"),
                      "classes": out}))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--nrhs", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--both", action="store_true", help="run the program and the stage tables (subprocesses)")
    a = ap.parse_args()
    if a.both:
        for mode in ("program", "stages"):
            env = dict(os.environ)
            if mode == "stages":
                env["PS_SOLVE"] = "stages"
            subprocess.run([sys.executable, __file__, "--config", a.config, "--nrhs", str(a.nrhs), "--reps",
                            str(a.reps)], env=env)
    else:
        run(a)
