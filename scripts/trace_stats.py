"""Summarise a program trace written by scripts/trace_prog.py:
  python scripts/trace_stats.py gpurun_out/trace_prog.npz [--bin-us 5]
Prints the busy/waiting CTA profile over time and the tasks whose completion
gates the longest idle stretches (the critical path of the dataflow program)."""
import argparse

import numpy as np


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--bin-us", type=float, default=5.0)
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    tr = np.load(a.path)["prog"].astype(np.int64)
    if len(tr) == 0:
        print("empty trace")
        return
    t0 = tr[:, 2].min()
    f, r, c, d = (tr[:, k] - t0 for k in (2, 3, 4, 5))
    task, nch, klen = tr[:, 8], tr[:, 12], tr[:, 13]
    s0, s1 = tr[:, 6], tr[:, 7]
    T = d.max()
    nsm = len(np.unique(tr[:, 1]))
    print(f"items {len(tr)}  span {T / 1e3:.1f} us  SMs {nsm}")
    wait, comp, fin = (r - f).sum(), (c - r).sum(), (d - c).sum()
    tot = wait + comp + fin
    print(f"item time: wait {wait / tot:.2%}  compute {comp / tot:.2%}  combine/finalise {fin / tot:.2%}")
    if (s0 > 0).all():
        prep = (s1 - s0) / 1e3
        lag = (tr[:, 2] - s1) / 1e3
        print(f"scheduler prep (ticket -> slot handed over) us: p10/50/90/99 = "
              f"{np.percentile(prep, [10, 50, 90, 99]).round(2)}, mean {prep.mean():.2f}")
        print(f"slot handed over -> compute warps start us: p10/50/90 = {np.percentile(lag, [10, 50, 90]).round(2)}; "
              f"items whose compute warps waited on the scheduler (< 0.2 us): {(lag < 0.2).mean():.1%}")
        print(f"item k-length: p10/50/90 = {np.percentile(klen, [10, 50, 90])}, mean {klen.mean():.0f}")
    b = a.bin_us * 1e3
    nb = int(T // b) + 1
    busy = np.zeros(nb)
    waiting = np.zeros(nb)
    for lo, hi, acc in ((r, c, busy), (f, r, waiting)):
        for x0, x1 in zip(lo, hi):
            i0, i1 = int(x0 // b), int(x1 // b)
            if i0 == i1:
                acc[i0] += (x1 - x0) / b
            else:
                acc[i0] += (b * (i0 + 1) - x0) / b
                acc[i0 + 1:i1] += 1
                acc[i1] += (x1 - b * i1) / b
    print(f"\n{'t(us)':>8} {'computing':>10} {'waiting':>8}")
    for i in range(nb):
        print(f"{i * a.bin_us:8.1f} {busy[i]:10.1f} {waiting[i]:8.1f}")
    # per task: first fetch, last ready, last done, items, k
    order = np.argsort(task, kind="stable")
    ts, idx = np.unique(task[order], return_index=True)
    rows = []
    for j, t in enumerate(ts):
        sl = order[idx[j]: idx[j + 1] if j + 1 < len(idx) else len(order)]
        rows.append((int(t), len(sl), f[sl].min(), r[sl].max(), d[sl].max(), int(klen[sl].sum()), int(nch[sl].max())))
    rows.sort(key=lambda x: x[4])
    # tasks with the longest wait-to-done (candidates for the critical path)
    print(f"\ntasks {len(rows)}; longest ready->done spans:")
    rows_span = sorted(rows, key=lambda x: -(x[4] - x[3]))[: a.top]
    print(f"{'task':>7} {'items':>6} {'fetch':>8} {'ready':>8} {'done':>8} {'span':>7} {'k':>8} {'nch':>4}")
    for t, n, ff, rr, dd, k, nc in rows_span:
        print(f"{t:7d} {n:6d} {ff / 1e3:8.1f} {rr / 1e3:8.1f} {dd / 1e3:8.1f} {(dd - rr) / 1e3:7.1f} {k:8d} {nc:4d}")
    # completion profile: done times of tasks by decile
    dn = np.array([x[4] for x in rows]) / 1e3
    print("\ntask completion percentiles (us):", np.percentile(dn, [10, 25, 50, 75, 90, 99, 100]).round(1))


if __name__ == "__main__":
    main()
