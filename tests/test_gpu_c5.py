"""BASELINE config 4 (PEC sphere r = 3 m, icosphere sub-7, N = 491520) on the GPU.

1. GPU vs oracle: tests/golden/C5_x.npz holds the oracle's two-term x for 2 RHS columns,
   written by scripts/c5_golden.py (oracle/ only: sequential scaling Eqs. 14-23 with
   the alpha panels spilled to disk, two-term solve Eqs. 24-36). This test regenerates
   C5 with the same seeded generator, requires the .hm file's stored section checksums
   to equal the golden's (bit-identical operator), and compares ps_solve per column at
   <= 1e-11 relative L2 — both as a 2-column solve (narrow tiles) and inside the bench's
   256-column launch (wide tiles).
2. Residual pins (properties that hold at any size), with the file's own
   near field on the host (numpy block mat-vec, independent of libps):
     * y0 = R D^-1 R^T b (GPU, ps_apply) solves the near field:  Z_N y0 = b;
     * x  = the two-term solution (ps_solve) satisfies        Z_N x  = b - Z_F y0
       (x = Z_N^-1 b - Z_N^-1 Z_F Z_N^-1 b, Appendix B of SURVEY.md), to rounding.

Generation takes ~7 min on the GPU box's 16 cores and ~40 GB of host memory.
"""
import os
import warnings

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "C5_x.npz")
TOL = 1e-11


def _near_apply(H, x):
    """Z_N x for RWG-ordered x (N x nrhs), from the file's symmetric near blocks."""
    xm = x[H.perm]                        # Morton order
    ym = np.zeros_like(xm)
    off = H.leaf_off
    for i, j, Z in H.near:
        a0, a1, b0, b1 = off[i], off[i + 1], off[j], off[j + 1]
        ym[a0:a1] += Z @ xm[b0:b1]
        if i != j:
            ym[b0:b1] += Z.T @ xm[a0:a1]
    y = np.empty_like(ym)
    y[H.perm] = ym
    return y


def test_near_apply_is_the_near_field(cfgdata):
    """The host Z_N mat-vec used below equals the dense near field (C1, CPU)."""
    from oracle import read_hm
    from oracle.dense import dense_ZN
    H = read_hm(cfgdata("C1")["hm"])
    rng = np.random.default_rng(0)
    x = rng.standard_normal((H.N, 2)) + 1j * rng.standard_normal((H.N, 2))
    ZN = dense_ZN(H)
    assert np.linalg.norm(_near_apply(H, x) - ZN @ x) <= 1e-13 * np.linalg.norm(ZN @ x)


def test_c5_golden_is_consistent():
    """CPU check of the committed golden: the oracle's x for C5 columns 0 and 127 (shape,
    finiteness, the recorded norms and the Eq. 45 ratios it implies)."""
    if not os.path.exists(GOLDEN):
        pytest.skip("tests/golden/C5_x.npz not generated (scripts/c5_golden.py)")
    g = np.load(GOLDEN)
    assert g["x"].shape == (491520, 2) and np.isfinite(g["x"]).all()
    assert list(g["cols"]) == [0, 127] and len(g["hm_checksums"]) == 9
    assert (g["it0"] > 0).all() and (g["it1"] > 0).all()


_state = {}


def _c5():
    if "h" not in _state:
        from hmgen.build import load_or_generate, read_rhs
        from paper_2109_04129_b200 import PsHandle
        from tests import _prefetch
        _prefetch.wait()                  # the generator child started at collection, if any
        meta = load_or_generate("C5")
        B, _ = read_rhs(meta["rhs"])
        h = PsHandle(meta["hm"])
        h.setup()
        _state.update(meta=meta, B=B, h=h)
    return _state


def _dev(A):
    import torch
    return torch.from_numpy(np.ascontiguousarray(np.asfortranarray(A).T)).cuda().T


def _host(T):
    return np.asfortranarray(T.T.cpu().numpy().T)


@pytest.mark.gpu
@pytest.mark.slow
def test_c5_vs_oracle_golden():
    pytest.importorskip("torch")
    import torch
    assert os.path.exists(GOLDEN), "tests/golden/C5_x.npz missing (scripts/c5_golden.py)"
    g = np.load(GOLDEN)
    st = _c5()
    import sys
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    from c5_golden import hm_checksums
    assert hm_checksums(st["meta"]["hm"]) == [str(s) for s in g["hm_checksums"]], \
        "regenerated C5 differs from the file the golden was computed on"
    cols = [int(c) for c in g["cols"]]
    ref = g["x"]
    h, B = st["h"], st["B"]
    # (a) the golden columns as one 2-column solve (narrow tiles)
    Bd = _dev(B[:, cols])
    Xd = torch.empty_like(Bd)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _, rep = h.solve(Bd, Xd)
    x = _host(Xd)
    err = np.linalg.norm(x - ref, axis=0) / np.linalg.norm(ref, axis=0)
    print(f"C5 vs oracle (2 columns): {err}")
    assert err.max() <= TOL, err
    assert np.allclose(rep["it0"], g["it0"], rtol=1e-11) and np.allclose(rep["it1"], g["it1"], rtol=1e-10)
    # (b) inside the bench's 256-column launch (wide tiles)
    Bd = _dev(B)
    Xd = torch.empty_like(Bd)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h.solve(Bd, Xd)
    x = Xd[:, cols].cpu().numpy()
    err = np.linalg.norm(x - ref, axis=0) / np.linalg.norm(ref, axis=0)
    print(f"C5 vs oracle (in the 256-column launch): {err}")
    assert err.max() <= TOL, err
    del Bd, Xd
    torch.cuda.empty_cache()


@pytest.mark.gpu
@pytest.mark.slow
def test_c5_residual_pins():
    pytest.importorskip("torch")
    import torch
    from oracle import read_hm
    from paper_2109_04129_b200 import PS_OP_DINV, PS_OP_R, PS_OP_RT, PS_OP_ZF
    from tests.conftest import rel_l2_cols
    st = _c5()
    h = st["h"]
    B = np.asfortranarray(st["B"][:, :2])
    Bd = _dev(B)
    Xd = torch.empty_like(Bd)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h.solve(Bd, Xd)
    t1, t2, y0 = torch.empty_like(Bd), torch.empty_like(Bd), torch.empty_like(Bd)
    h.apply(PS_OP_RT, Bd, t1)
    h.apply(PS_OP_DINV, t1, t2)
    h.apply(PS_OP_R, t2, y0)
    tF = torch.empty_like(Bd)
    h.apply(PS_OP_ZF, y0, tF)
    x, y0h, tFh = _host(Xd), _host(y0), _host(tF)
    hm = st["meta"]["hm"]
    h.close()
    _state.clear()
    H = read_hm(hm, mmap=True)
    r0 = rel_l2_cols(_near_apply(H, y0h), B)
    r1 = np.linalg.norm(_near_apply(H, x) - (B - tFh), axis=0) / np.linalg.norm(B, axis=0)
    print(f"C5 N={H.N}: ||Z_N y0 - b||/||b|| = {r0.max():.3e}, ||Z_N x - (b - Z_F y0)||/||b|| = {r1.max():.3e}")
    assert r0.max() <= 1e-9, r0
    assert r1.max() <= 1e-9, r1
