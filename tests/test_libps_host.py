"""libps host-side checks that need no GPU: the library builds for sm_100a,
loads, exports every symbol include/ps.h declares, rejects bad files with the
documented statuses, and its symbolic analysis (struct(k) with fill) agrees
with the fill the oracle discovers while eliminating (Eq. 21)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2109_04129_b200 import binding
from paper_2109_04129_b200.binding import INFO_KEYS, load_library

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    txt = open(os.path.join(ROOT, "include", "ps.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b([a-z_]+)\s*\(", txt)) - {"if", "sizeof"})


def test_library_exports_every_declared_symbol():
    L = load_library()
    syms = _declared_symbols()
    assert {"hm_load", "ps_setup", "ps_solve", "ps_free", "ps_n", "ps_last_error"} <= set(syms)
    for s in syms:
        assert hasattr(L, s), f"libps.so does not export {s}"


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", binding.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _analyze(path):
    L = load_library()
    out = (ctypes.c_double * len(INFO_KEYS))()
    n = L.ps_analyze(path.encode(), out, len(INFO_KEYS))
    if n < 0:
        return -n, L.ps_last_error(None).decode()
    return 0, {k: out[i] for i, k in enumerate(INFO_KEYS[:n])}


def test_bad_files(tmp_path, synthfile):
    st, msg = _analyze(str(tmp_path / "missing.hm"))
    assert st == binding.PS_EIO
    p, _ = synthfile(n_points=150, seed=1)
    raw = bytearray(open(p, "rb").read())
    q = tmp_path / "magic.hm"
    q.write_bytes(b"XXXX" + bytes(raw[4:]))
    assert _analyze(str(q))[0] == binding.PS_EFORMAT
    raw2 = bytearray(raw)
    raw2[len(raw2) // 2] ^= 1
    q2 = tmp_path / "flip.hm"
    q2.write_bytes(bytes(raw2))
    st, msg = _analyze(str(q2))
    assert st == binding.PS_EFORMAT and "checksum" in msg
    q3 = tmp_path / "trunc.hm"
    q3.write_bytes(bytes(raw[: len(raw) - 100]))
    assert _analyze(str(q3))[0] == binding.PS_EFORMAT


def test_null_arguments():
    L = load_library()
    h = ctypes.c_void_p()
    assert L.hm_load(None, None, ctypes.byref(h)) == binding.PS_EINVAL
    assert L.ps_n(None) == -1
    assert L.ps_setup(None, None) == binding.PS_EINVAL
    assert L.ps_solve(None, 1, None, 1, None, 1, 1, None, None) == binding.PS_EINVAL
    assert L.ps_solve_series(None, None, 1, None, 1, None, 1, 1, None, None) == binding.PS_EINVAL
    assert L.ps_solve_async(None, 1, None, 1, None, 1, None) == binding.PS_EINVAL
    assert L.ps_solve_report(None, None) == binding.PS_EINVAL
    L.ps_free(None)                     # NULL-safe


@pytest.mark.parametrize("case", ["C1", "T2", "synth"])
def test_symbolic_fill_matches_oracle(case, cfgdata, synthfile):
    """libps's symbolic struct(k) (union over elimination-tree children) must
    give exactly the alpha blocks the oracle creates while eliminating."""
    from oracle import compute_scaling, read_hm
    path = cfgdata(case)["hm"] if case != "synth" else synthfile(n_points=500, seed=3, clustered=True)[0]
    st, info = _analyze(path)
    assert st == 0, info
    S = compute_scaling(read_hm(path))
    blocks = sum(len(a) for a in S.alpha)
    nR = sum(S.sizes[k] * sum(S.sizes[j] for j in S.alpha[k]) for k in range(S.n))
    nD = sum(int(s) ** 2 for s in S.sizes)
    assert info["alpha_blocks"] == blocks
    assert info["nR"] == nR
    assert info["nD"] == nD
    assert info["N"] == S.N


def _chains_from_oracle(S, tmax=4096):
    """Chain pieces of the elimination tree, written from the definition
    (DESIGN.md §6): maximal paths p -> parent(p) whose upper nodes have a single
    child, cut before exceeding tmax unknowns. Returns (pieces, chain-graph height)."""
    n = S.n
    st = [sorted(S.alpha[k].keys()) for k in range(n)]
    par = [s[0] if s else -1 for s in st]
    nchild = [0] * n
    for p in range(n):
        if par[p] >= 0:
            nchild[par[p]] += 1
    cid = [-1] * n
    pieces = []
    for p in range(n):
        if cid[p] >= 0:
            continue
        c, U, q = [p], int(S.sizes[p]), p
        while par[q] >= 0 and nchild[par[q]] == 1 and cid[par[q]] < 0 and U + int(S.sizes[par[q]]) <= tmax:
            q = par[q]
            c.append(q)
            U += int(S.sizes[q])
        for x in c:
            cid[x] = len(pieces)
        pieces.append(c)
    height = [0] * len(pieces)
    for i in sorted(range(len(pieces)), key=lambda i: pieces[i][-1]):
        up = par[pieces[i][-1]]
        if up >= 0:
            j = cid[up]
            assert pieces[j][0] == up          # a piece's top hangs below another piece's first node
            height[j] = max(height[j], height[i] + 1)
    return pieces, max(height) + 1


@pytest.mark.parametrize("case", ["C1", "T2", "synth"])
def test_chain_pieces_match_definition(case, cfgdata, synthfile):
    """The chain pieces libps collapses through T_c (ps_info) agree with the
    definition applied to the elimination tree the oracle discovers."""
    from oracle import compute_scaling, read_hm
    path = cfgdata(case)["hm"] if case != "synth" else synthfile(n_points=900, seed=7, clustered=True)[0]
    st, info = _analyze(path)
    assert st == 0, info
    S = compute_scaling(read_hm(path))
    pieces, height = _chains_from_oracle(S)
    multi = [c for c in pieces if len(c) >= 2]
    assert info["chains"] == len(multi)
    assert info["chain_height"] == height
    assert info["T_entries"] == sum(int(sum(S.sizes[p] for p in c)) ** 2 for c in multi)
    assert height < info["height"]           # collapsing chains shortens the dependency path


@pytest.mark.parametrize("P", [2, 4, 8])
def test_rank_share_of_device_memory(cfgdata, P):
    """Host-only per-rank analysis of the row partition (ps_analyze_rank): every rank
    holds less than the single-GPU operator (alpha panels, D^-1, T: far stacks stay
    whole) and less than the single-GPU setup arenas (near blocks, W, panels, D^-1);
    the interiors and the separators tile the unknowns."""
    from paper_2109_04129_b200.binding import analyze
    path = cfgdata("C2")["hm"]
    one = analyze(path)
    ranks = [analyze(path, g, P) for g in range(P)]
    assert sum(r["own_rows"] for r in ranks) + ranks[0]["sep_rows"] == one["N"]
    assert all(r["nranks"] == P for r in ranks)
    assert max(r["setup_bytes"] for r in ranks) < one["setup_bytes"]
    assert max(r["op_bytes"] for r in ranks) < one["op_bytes"]
    if P >= 4:                                   # the separators are a minority of the setup
        assert max(r["setup_bytes"] for r in ranks) < 0.75 * one["setup_bytes"]


@pytest.mark.parametrize("name,nrhs", [("C1", 1), ("C1", 9), ("C1", 70), ("T2", 181), ("C2", 1), ("C2", 181),
                                       ("C3", 1), ("C4", 360)])
def test_solve_program_is_race_and_deadlock_free(cfgdata, name, nrhs):
    """ps_validate (host-only) on the exact tables ps_solve launches: every operand
    access inside its arena; every pair of tasks writing one workspace element, and
    every reader / writer pair of a range, ordered by the dependency graph
    (happens-before) — no data race; every item's producers at smaller tickets —
    no deadlock of the persistent kernel. (compute-sanitizer is closed on this
    pool: this is the race / bounds evidence for the dataflow program.)"""
    from paper_2109_04129_b200.binding import validate
    r = validate(cfgdata(name)["hm"], nrhs)
    assert r["items"] > 0 and r["read_ranges"] >= r["segments"]


def test_solve_program_edge_cases_validate(synthfile):
    from paper_2109_04129_b200.binding import validate
    for kw in (dict(n_points=300, seed=1, clustered=True), dict(n_points=40, seed=2)):
        path = synthfile(**kw)[0]
        for nrhs in (1, 8, 64, 65):
            validate(path, nrhs)


def test_far1p_tables_validate(cfgdata):
    """nrhs <= 8: the program is two launches around the far1p apply; both the program and
    the far1p tables pass the checker, also with small items (many big-block chunks)."""
    import subprocess
    import sys
    path = cfgdata("C1")["hm"]
    for env in ({"PS_FAR1P": "1"}, {"PS_FAR1P": "1", "PS_F1P_CHUNK": "64"}):
        code = ("from paper_2109_04129_b200.binding import validate\n"
                f"v = validate({path!r}, 1)\n"
                "assert v['far1p_items'] and v['far1p_items'] > 0, v\n"
                f"assert validate({path!r}, 64)['far1p_items'] is None\n"
                "print(v['far1p_items'])\n")
        r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stderr[-800:]


@pytest.mark.parametrize("brk,what", [(1, "unordered"), (2, "precedes"), (3, "outside its region"),
                                      (4, "out of order"), (5, "outside the FB arena")])
def test_validator_catches_broken_tables(cfgdata, brk, what):
    """The checker itself: a dropped dependency, an item moved before its producer,
    an operator offset outside its region, a far1p consumer moved before its producers
    and a far1p item outside the FB arena are each reported."""
    import subprocess
    import sys
    path = cfgdata("C1")["hm"]
    code = ("from paper_2109_04129_b200.binding import validate\n"
            f"validate({path!r}, 1)\n")
    env = dict(os.environ, PS_VALIDATE_BREAK=str(brk), PS_FAR1P="1", PS_F1P_CHUNK="64")   # 64: big far1p blocks
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and what in r.stderr, r.stderr[-500:]
