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
