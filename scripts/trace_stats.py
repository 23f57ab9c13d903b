"""Summarise a trace_flow.py capture (per-item timing of the dataflow kernel)."""
import sys
import numpy as np
d = np.load(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/trace_C2.npz')
for nm in ['fwd', 'bwd', 'dinv', 'far1', 'far2']:
    tr = d[nm].astype(np.float64)
    t0 = tr[:, 2].min()
    f, r, c, e = [(tr[:, j] - t0) / 1e3 for j in (2, 3, 4, 5)]
    wait, comp, pub = r - f, c - r, e - c
    klen = tr[:, 11]
    ks = np.ceil(klen / 16)
    m = ks > 0
    T = np.linspace(0, e.max(), 10)
    busy = [int(((r <= t) & (c > t)).sum()) for t in T]
    print(f"{nm:5s} items {len(tr):6d} span {e.max():7.0f}us wait {wait.mean():6.1f} comp {comp.mean():6.2f} "
          f"pub {pub.mean():5.2f} us/kstep {np.median(comp[m] / ks[m]):.3f} ksteps {ks.sum():.0f} busy {busy}")
