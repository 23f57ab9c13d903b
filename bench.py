#!/usr/bin/env python
"""bench.py — ps_solve throughput (N*nrhs/s, complex128) of libps on B200.

One "step" = one ps_solve of the configured right-hand-side block: the whole
two-term hot path of SURVEY.md §8(a) rows a4-a8 (forward sweep R^T + D^-1,
backward sweep R, far field Z_F, forward sweep + D^-1, combine + norms,
backward sweep), device-resident B and X. The O(N) setup (rows a1-a3) is run
once before the timed region and reported separately as `setup_ms`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Default workload: C4 (BASELINE configs[3], the largest config that fits one GPU's
measurement budget: cylinder, N = 96000, 360 RHS), plus the same handle at nrhs = 1
in the line's "nrhs1" object (the HBM-bound half of the metric).

Multi-GPU (torchrun, one process per GPU): with >= 16 columns per rank the config's
RHS block is split into distinct column blocks (replicated operator, no data-path
collective; `scaling: strong`); with fewer (nrhs = 1) the operator is row-partitioned
over the ranks with NCCL exchanges. Time = max over ranks.

--impl reference runs the CPU oracle (oracle/, numpy complex128) on the host
cores as the reference arm (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ps_solve N·nrhs/sec (complex128)"
UNIT = "N·nrhs/s"
SM_COUNT = 148
DFMA_PER_SM_PER_CLK = 64          # FP64 FMA lanes per SM (B200); 2 flop each


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = {}
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
    return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region:
    one nvidia-smi process in loop mode (a sample every 20 ms), each line
    time-stamped on arrival; mark() / stop() bracket the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.samples = []
        self._all = []
        self._p = None
        self._t = None
        self.t0 = self.t1 = None

    def _read(self):
        for line in self._p.stdout:
            if line.strip():
                self._all.append((time.perf_counter(), [x.strip() for x in line.split(",")]))

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "20"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            t = time.perf_counter()
            while not self._all and time.perf_counter() - t < 3.0:   # sampler is live
                time.sleep(0.01)
        except Exception:
            self._p = None
        return self

    def mark(self):
        self.t0 = time.perf_counter()

    def stop(self):
        self.t1 = time.perf_counter()

    def __exit__(self, *a):
        if self._p is None:
            return
        if self.t1 is None:
            self.t1 = time.perf_counter()
        time.sleep(0.05)
        self._p.terminate()
        try:
            self._p.wait(timeout=10)
        except Exception:
            self._p.kill()
        if self._t:
            self._t.join(timeout=5)
        t0 = self.t0 if self.t0 is not None else 0.0
        inside = [v for (t, v) in self._all if t0 <= t <= self.t1]
        if not inside and self._all:      # region shorter than one sample period: nearest sample
            inside = [min(self._all, key=lambda tv: abs(tv[0] - 0.5 * (t0 + self.t1)))[1]]
        self.samples = inside

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


_ORACLE_CACHE = {}


def _oracle_state(meta):
    """(H, S) of the oracle for this config, computed once per process (the reference
    arm's steps time the solve on the cached scaling)."""
    from oracle import compute_scaling, read_hm
    key = meta["hm"]
    if key not in _ORACLE_CACHE:
        H = read_hm(meta["hm"])
        t0 = time.perf_counter()
        S = compute_scaling(H)
        _ORACLE_CACHE[key] = (H, S, time.perf_counter() - t0)
    return _ORACLE_CACHE[key]


def _cores():
    try:
        from threadpoolctl import threadpool_info
        return int(max([d.get("num_threads", 1) for d in threadpool_info()] + [1]))
    except Exception:
        return os.cpu_count()


def cpu_oracle_arm(meta, B, seconds=12.0, max_cols=16):
    """The oracle (as it stands) on a bounded sample: the first `max_cols` RHS columns,
    solved repeatedly until ~`seconds` of CPU work (the oracle's scaling, computed once
    per process, is excluded). Returns (N*nrhs/s, details)."""
    from oracle import solve
    H, S, t_setup = _oracle_state(meta)
    cols = B[:, :max_cols]
    n_done = 0
    t0 = time.perf_counter()
    while True:
        solve(H, S, cols)
        n_done += cols.shape[1]
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    v = H.N * n_done / el
    return v, dict(cores=_cores(), t_setup_s=t_setup, solved_cols=n_done, seconds=el,
                   sample=f"the first {cols.shape[1]} of the workload's {B.shape[1]} RHS columns, solved "
                          f"repeatedly for {el:.1f} s (oracle scaling, {t_setup:.1f} s once per process, "
                          f"excluded)")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from hmgen.build import load_or_generate, read_rhs
    meta = load_or_generate(args.config)
    B, _ = read_rhs(meta["rhs"])
    nrhs = args.nrhs or B.shape[1]
    if nrhs > B.shape[1]:
        B = np.tile(B, (1, -(-nrhs // B.shape[1])))
    B = np.asfortranarray(B[:, :nrhs])
    vals = []
    det = None
    for s in range(args.warmup + args.steps):
        secs = args.ref_seconds or max(2.0, min(20.0, 60.0 / max(1, args.steps)))
        v, det = cpu_oracle_arm(meta, B, seconds=secs, max_cols=min(nrhs, 16))
        if s >= args.warmup:
            vals.append(v)
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * meta["N"] * nrhs / v, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": _config(args, meta, nrhs, 1),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": det["cores"], "kind": "oracle",
                             "sample": det["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def _ncu_traffic(config, nrhs):
    """Mean DRAM bytes (read + write) per flow_kernel launch of one solve, from the committed
    ncu --set full summary of this config (profiles/*/ncu_full_<cfg>_<nrhs>_*.json, written by
    scripts/ncu_summary.py) — only when it was captured on the build this run uses (same libps
    source hash); else (None, reason)."""
    import glob
    from paper_2109_04129_b200.build import source_hash
    cur = source_hash()
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", f"ncu_full_{config}_{nrhs}_*.json")),
                   key=os.path.getmtime)
    for fn in reversed(files):
        try:
            with open(fn) as f:
                d = json.load(f)
        except Exception:
            continue
        if not isinstance(d, dict) or d.get("src_hash") != cur:
            continue

        def mb(v):
            x, u = v.split()
            return float(x) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        # the capture holds ONE solve (scripts/ncu_solve.py): its dataflow-program launch(es) and,
        # for nrhs <= 8, the far1p apply — the DRAM bytes of that kernel chain
        vals = [mb(r["dram__bytes_read.sum"]) + mb(r["dram__bytes_write.sum"]) for r in d["rows"]
                if any(k in r.get("Kernel Name", "") for k in ("flow_kernel", "far1p", "far_reduce"))]
        if vals:
            return sum(vals), os.path.relpath(fn, ROOT)
    return None, f"no committed ncu --set full capture of {config}-{nrhs} on this build (libps {cur})"


def _config(args, meta, nrhs, world):
    rows = getattr(args, "mode", "cols") == "rows" and world > 1
    return {"workload": f"{args.config}-{nrhs}: {meta['desc']}", "N": meta["N"],
            "nrhs_per_gpu": nrhs, "global_nrhs": getattr(args, "nrhs_global", nrhs),
            "n_leaves": meta["n_leaves"],
            "queueing": ("value / nrhs1: the K timed solves queued back to back with ps_solve_async (all "
                         "kernels of every step incl. the Eq. 44-45 norms; no host synchronisation between "
                         "steps), the last solve's report read with ps_solve_report before the closing "
                         "synchronisation; e2e: synchronous ps_solve per step (host buffers, full report)"),
            "parallelism": (f"row partition x{world} (elimination-tree subtrees per rank, replicated "
                            f"separators; NCCL all-reduce of separator rows, all-gather of w and x)"
                            if rows else f"rhs-columns x{world} (replicated operator, distinct columns per "
                                         f"rank, no data-path collective)"),
            "l2": ("host oracle (no GPU L2)" if not hasattr(args, "op_mb") else
                   f"operator {getattr(args, 'op_mb', 0):.0f} MB < 2 x the 126 MB L2: a 256 MB buffer is "
                   "written before every timed step (per-step CUDA events exclude it)"
                   if getattr(args, "flush", False) else
                   f"operator (alpha panels + D^-1 + far factors + T) = {getattr(args, 'op_mb', 0):.0f} MB "
                   "exceeds the 126 MB L2; no flush")}


FP64_PEAK = 37.02   # TF/s: measured on this pool's B200 (scripts/fp64_peak.cu, profiles/r1/fp64_peak_b200.json)


def _time_solves(h, Bd, Xd, st, steps, flush_buf, dist, world):
    """Device ms per solve over `steps` timed solves (CUDA events on the solve stream). The
    solves are queued with ps_solve_async (every kernel of the step, the Eq. 44-45 norms
    included, no host synchronisation between steps); the report of the last one is read
    back (ps_solve_report) before the closing synchronisation. Row-partition handles
    (NCCL) keep the synchronous ps_solve."""
    import torch
    sync_only = not Bd.is_cuda or (world > 1 and getattr(h, "partitioned", False))

    def step():
        if sync_only:
            h.solve(Bd, Xd, stream=st, want_norms=False)
        else:
            h.solve_async(Bd, Xd, stream=st)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("timed")        # ncu --nvtx --nvtx-include "timed/" selects these launches
    if flush_buf is not None:                  # per-step events, L2 written between steps
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a_, b_ in evs:
            flush_buf.fill_(1)
            a_.record(st)
            step()
            b_.record(st)
        if not sync_only:
            h.solve_report()
        torch.cuda.synchronize()
        ms = sum(a_.elapsed_time(b_) for a_, b_ in evs) / steps
    else:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            step()
        e1.record(st)
        if not sync_only:
            h.solve_report()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
    torch.cuda.nvtx.range_pop()
    if world > 1:
        dist.barrier()
    return ms


def _roofline(h, Bd, Xd, st, nrhs, args, info, rep):
    """Roofline object of the dominant kernel (the one dataflow-program launch per solve):
    SURVEY §8(d)'s algorithmic work of one solve (rep: 8 nrhs (4 n_R + 2 n_D + 2 n_F) flop;
    16 (4 n_R + 2 n_D + n_F) + 16 * 12 N nrhs bytes) / that kernel's mean launch time, timed
    with CUDA events on the launching stream (ps_profile)."""
    steps = max(1, args.profile_steps)
    h.profile(True)
    for _ in range(steps):
        h.solve(Bd, Xd, stream=st, want_norms=False)
    prof = h.profile_read()
    h.profile(False)
    # the dominant kernel chain of one solve: the dataflow program (one launch; for nrhs <= 8 two
    # launches around the one-pass far apply, whose kernels are the far1p class)
    f1p = prof.get("far1p", {"ms": 0.0, "launches": 0, "flops": 0.0, "bytes": 0.0})
    chain_ms = (prof["solve_program"]["ms"] + f1p["ms"]) / steps
    k_ms = chain_ms
    tot_ms = sum(prof[c]["ms"] for c in prof) / steps
    exe_fl = (prof["solve_program"]["flops"] + f1p["flops"]) / steps
    exe_by = (prof["solve_program"]["bytes"] + f1p["bytes"]) / steps
    peaks = _peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6548.2))
    alg_fl, alg_by = rep["flops"], rep["bytes"]
    traffic, traffic_src = _ncu_traffic(args.config, nrhs)
    if nrhs <= 8:
        gbs = alg_by / (k_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)"}
    else:
        tf = alg_fl / (k_ms * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": tf, "peak": FP64_PEAK, "unit": "TFLOP/s", "frac": tf / FP64_PEAK,
                "peak_source": ("FP64 (DFMA and mma.sync f64 share one pipe budget; tcgen05 has no f64 kind): "
                                "measured 37.02 TF on this pool's B200 (profiles/r1/fp64_peak_b200.json) = "
                                "148 SM x 64 FP64 FMA/clk x 2 flop x 1.965 GHz (37.2 TF derived); "
                                "MEASURED_PEAKS.json has no FP64 entry"),
                # the tensor-core consumer forms each complex product with Gauss's three real
                # multiplications, so the algorithmic complex rate (8 flop per
                # complex multiply-add) can reach 4/3 of the real FP64 peak
                "complex_3m_peak": FP64_PEAK * 4.0 / 3.0,
                "frac_of_complex_3m_peak": tf / (FP64_PEAK * 4.0 / 3.0)}
    roof.update({
        "traffic": traffic, "traffic_source": traffic_src,
        "algorithmic_per_launch": {"flop": alg_fl, "bytes": alg_by,
                                   "formula": "SURVEY 8(d): flop = 8 nrhs (4 n_R + 2 n_D + 2 n_F); bytes = "
                                              "16 (4 n_R + 2 n_D + n_F) + 16 x 12 N nrhs"},
        "executed_per_launch": {"flop": exe_fl, "bytes": exe_by,
                                "note": "products the kernel's task tables execute: chain-internal alpha "
                                        "blocks replaced by the T_c products (DESIGN.md R23), operator "
                                        "bytes only"},
        "executed_over_algorithmic_operator_bytes": exe_by / (16.0 * (4 * info["nR"] + 2 * info["nD"] + info["nF"])),
        "kernel": ("ps::flow_kernel_ws x2 (sweeps before / after the far field) + ps::far1p_kernel and "
                   "far_reduce (one-pass far apply, DESIGN.md §6): device time per solve"
                   if f1p["launches"] else
                   "ps::flow_kernel / flow_kernel_ws (persistent dataflow gather-GEMM: the whole two-term "
                   "solve as one launch)"),
        "kernel_ms_per_launch": k_ms,
        "kernel_parts_ms": {"solve_program": prof["solve_program"]["ms"] / steps, "far1p": f1p["ms"] / steps},
        "kernel_share_of_step": chain_ms / tot_ms if tot_ms > 0 else None})
    return roof


def _next_rows(h, Bd, Xd, st, args, info, N, terms=4, steps=3):
    """SURVEY 8(f) NEXT-3 / NEXT-4 on the bench's handle and RHS block (CUDA events on the
    solve stream, after one warm-up call each): ps_solve_series at 2 and `terms` terms
    (per extra term = one U application: 16 (2 n_R + n_D + n_F) bytes, 8 nrhs (2 n_R + n_D +
    2 n_F) flop), and the monostatic RCS sweep (ps_farfield, direction c = the backscatter of
    incidence c) of the solve's currents."""
    import torch
    from hmgen.build import CONFIGS, make_mesh, plane_wave_dirs, rwg_basis
    from paper_2109_04129_b200 import farfield

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    R = Bd.shape[1]
    out = {}
    t2 = timed(lambda: h.solve_series(Bd, Xd, max_terms=2, stream=st))
    tn = timed(lambda: h.solve_series(Bd, Xd, max_terms=terms, stream=st))
    _, rep = h.solve_series(Bd, Xd, max_terms=terms, stream=st)
    tt = (tn - t2) / (terms - 2)
    nR, nD, nF = info["nR"], info["nD"], info["nF"]
    by = 16.0 * (2 * nR + nD + nF) + 16.0 * 6 * N * R
    fl = 8.0 * R * (2 * nR + nD + 2 * nF)
    peaks = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6548.2))
    out["series"] = {"row": "NEXT-3 n-term series (ps_solve_series)", "terms": terms,
                     "ms_terms_2": t2, f"ms_terms_{terms}": tn, "ms_per_extra_term": tt,
                     "value": N * R * terms / (tn * 1e-3), "unit": "N*nrhs*terms/s",
                     "per_term_roofline": ({"bound": "hbm", "achieved": by / (tt * 1e-3) / 1e9, "peak": hbm,
                                            "unit": "GB/s", "frac": by / (tt * 1e-3) / 1e9 / hbm}
                                           if R <= 8 else
                                           {"bound": "alu", "achieved": fl / (tt * 1e-3) / 1e12, "peak": FP64_PEAK,
                                            "unit": "TFLOP/s", "frac": fl / (tt * 1e-3) / 1e12 / FP64_PEAK}),
                     "last_ratio_max": float((rep["it_norm"][-1] / rep["it_norm"][-2]).max()),
                     "launches": int(rep["launches"])}
    name = args.config
    if name in CONFIGS and R == len(plane_wave_dirs(CONFIGS[name])[1]):
        cfg = CONFIGS[name]
        m = make_mesh(cfg)
        bs = rwg_basis(m)
        _, khat, _ = plane_wave_dirs(cfg)
        g = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (m.nodes, m.tris, bs.tp, bs.tm, bs.vp, bs.vm)]
        rh = torch.from_numpy(-np.asarray(khat)).cuda()
        h.solve(Bd, Xd, stream=st, want_norms=False)
        eta = 120 * np.pi
        tr = timed(lambda: farfield(*g, cfg.k, eta, Xd, rh, mono=True, stream=st))
        pairs = R * 14 * bs.N
        out["rcs"] = {"row": "NEXT-4 monostatic RCS sweep (ps_farfield)", "directions": R, "ms": tr,
                      "value": pairs / (tr * 1e-3), "unit": "direction-sample pairs/s",
                      "roofline": {"bound": "alu", "achieved": 26.0 * pairs / (tr * 1e-3) / 1e12, "peak": FP64_PEAK,
                                   "unit": "TFLOP/s", "frac": 26.0 * pairs / (tr * 1e-3) / 1e12 / FP64_PEAK,
                                   "note": "13 FMA per pair counted (phase 3, current x phase 4, 3 complex "
                                           "accumulations 6); the FP64 sincos per pair is not counted"}}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4",
                    help="BASELINE config (default C4: the largest single-GPU config, 360 RHS)")
    ap.add_argument("--nrhs", type=int, default=0, help="RHS columns (default: the config's full table)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nrhs1", action="store_true", help="skip the embedded nrhs = 1 (HBM-bound) measurement")
    ap.add_argument("--no-next", action="store_true",
                    help="skip the NEXT-3 (n-term series) / NEXT-4 (RCS) timings on the bench handle")
    ap.add_argument("--profile-steps", type=int, default=2)
    ap.add_argument("--ref-seconds", type=float, default=0.0,
                    help="--impl reference: seconds of oracle work per step (default: 60 s / steps, 2..20 s)")
    ap.add_argument("--flush-l2", default="auto", choices=["auto", "on", "off"],
                    help="write a 256 MB buffer before every timed step (auto: when the operator is "
                         "smaller than 2 x L2, e.g. C1)")
    ap.add_argument("--partition", default="auto", choices=["auto", "cols", "rows"],
                    help="N > 1: cols = replicated operator, the config's RHS block split into distinct "
                         "column blocks per rank (no collective); rows = row partition of the operator (NCCL "
                         "exchanges, every rank works on the whole block); auto = cols when nrhs >= 16 N, else rows")
    args = ap.parse_args()
    warnings.simplefilter("ignore", RuntimeWarning)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from hmgen.build import load_or_generate, read_rhs
    from paper_2109_04129_b200 import PsHandle
    from paper_2109_04129_b200.dist import column_slice, max_over_ranks

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:                      # NCCL's INIT lines (nranks, transports) stay on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        meta = load_or_generate(args.config)
    if world > 1:
        dist.barrier()
        if rank != 0:
            meta = load_or_generate(args.config)
    Bfull, _ = read_rhs(meta["rhs"])
    nrhs_global = args.nrhs or Bfull.shape[1]
    if nrhs_global > Bfull.shape[1]:        # more columns than the config's table: repeat it
        Bfull = np.tile(Bfull, (1, -(-nrhs_global // Bfull.shape[1])))
    mode = args.partition
    if mode == "auto":
        mode = "cols" if (world == 1 or nrhs_global >= 16 * world) else "rows"
    args.mode = mode
    args.nrhs_global = nrhs_global
    if mode == "rows":
        B = np.asfortranarray(Bfull[:, :nrhs_global])
    else:                                   # distinct columns per rank (strong split of the block)
        B = np.asfortranarray(Bfull[:, :nrhs_global][:, column_slice(nrhs_global, world, rank, "strong")])
    nrhs = B.shape[1]
    N = meta["N"]

    if mode == "rows" and world > 1:
        from paper_2109_04129_b200 import nccl_unique_id
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        h = PsHandle(meta["hm"], device=local, rank=rank, nranks=world, partition=True, nccl_id=obj[0])
        h.partitioned = True
    else:
        h = PsHandle(meta["hm"], device=local, rank=rank, nranks=world)
    # one non-default stream for everything timed: torch's ops, libps's launches (ps_solve /
    # ps_solve_async take its handle) and the CUDA events that bracket them
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.setup()
    setup_ms = 1e3 * (time.perf_counter() - t0)
    info = h.info()

    def dev(A):
        return torch.from_numpy(np.array(A.T, order="C")).cuda().T

    Bd = dev(B)
    Xd = torch.empty_like(Bd)
    args.op_mb = 16.0 * sum(float(info.get(k, 0.0)) for k in ("nR", "nD", "nF", "T_entries")) / 2**20
    args.flush = args.flush_l2 == "on" or (args.flush_l2 == "auto" and args.op_mb < 2 * 126)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if args.flush else None
    for _ in range(args.warmup):
        _, rep = h.solve(Bd, Xd, stream=st)
    with ClockSampler(local) as clk:
        clk.mark()
        step_ms = _time_solves(h, Bd, Xd, st, args.steps, flush_buf, dist, world)
        clk.stop()
    ms = max_over_ranks(step_ms, dist, "cuda")
    _, rep = h.solve(Bd, Xd, stream=st)
    launches = int(rep["launches"])
    ratio = rep["ratio"]

    # ---- end to end: host (pinned) buffers through the C ABI, copies inside ----
    Bh = torch.from_numpy(np.array(B.T, order="C")).pin_memory().T
    Xh = torch.empty((nrhs, N), dtype=torch.complex128).pin_memory().T
    for _ in range(max(1, args.warmup)):
        h.solve(Bh, Xh, stream=st, want_norms=False)
    ms_e2e = max_over_ranks(_time_solves(h, Bh, Xh, st, args.steps, None, dist, world), dist, "cuda")

    roof = _roofline(h, Bd, Xd, st, nrhs, args, info, rep)
    total_cols = nrhs_global
    value = N * total_cols / (ms * 1e-3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded EFIE H-matrix from hmgen; plane-wave RHS)",
            "config": _config(args, meta, nrhs, world),
            "setup_ms": setup_ms,
            "setup_tflops": 8.0 * info["setup_madds"] / (setup_ms * 1e-3) / 1e12,
            "structure": {k: info[k] for k in ("n_leaves", "alpha_blocks", "nR", "nD", "nF", "height", "depth",
                                               "T_entries")},
            "series": {"ratio_min": float(ratio.min()), "ratio_max": float(ratio.max()),
                       "n_diverged": int(rep["n_diverged"]),
                       "note": "ratio = ||it_1||/||it_0|| from the C ABI (Eq. 45); >= 0.1 flags divergence. "
                               "BASELINE configs use 0.25-lambda leaves, below the paper's 0.5-lambda accuracy "
                               "threshold (DESIGN.md R14)"},
            "roofline": roof,
            "e2e": {"value": N * total_cols / (ms_e2e * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": 16 * N * nrhs, "d2h_bytes_per_step": 16 * N * nrhs,
                    "ms_per_step": ms_e2e},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary()}

    # ---- nrhs = 1 (operator streaming, HBM-bound) on the same handle: the metric's other half ----
    if nrhs > 1 and not args.no_nrhs1 and mode == "cols":
        B1 = Bd[:, :1].contiguous()
        X1 = torch.empty_like(B1)
        for _ in range(args.warmup):
            _, rep1 = h.solve(B1, X1, stream=st)
        with ClockSampler(local) as clk1:
            clk1.mark()
            ms1 = max_over_ranks(_time_solves(h, B1, X1, st, args.steps, flush_buf, dist, world), dist, "cuda")
            clk1.stop()
        _, rep1 = h.solve(B1, X1, stream=st)
        roof1 = _roofline(h, B1, X1, st, 1, args, info, rep1)
        line["nrhs1"] = {"workload": f"{args.config}-1 (first column of the same block)",
                         "value": N * world / (ms1 * 1e-3), "unit": UNIT, "ms_per_step": ms1,
                         "roofline": roof1, "clocks": clk1.summary()}
    # ---- SURVEY 8(f) rows after the two-term solve, on the same handle and block ----
    if not args.no_next and mode == "cols" and world == 1:
        line["next_rows"] = _next_rows(h, Bd, Xd, st, args, info, N)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, det = cpu_oracle_arm(meta, B)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": det["cores"], "kind": "oracle",
                                "sample": det["sample"]}
    if rank == 0:
        print(json.dumps(line))
    h.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
