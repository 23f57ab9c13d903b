"""GPU parity of the n-term / adaptive power series (ps_solve_series; SURVEY §8(f) NEXT-3,
PAPER.md Eqs. 35-36, 44-45; stopping rule DESIGN.md R25) against the oracle
(oracle.series_solve / series_solve_adaptive): per column relative L2 <= 1e-11 for x,
per-term norms ||it_n|| to 1e-10, the same number of terms and the same divergence flags.
Cases: a convergent synthetic system (fixed n = 1, 2, 3, 7 and adaptive to the dense-LU
solution), ragged synthetic leaves, and C1 (two terms = ps_solve; four terms, diverging
ratio 0.8 at the first term)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from hmgen.synth import random_rhs                          # noqa: E402
from oracle import (apply_Dinv, apply_R, apply_Rt, apply_U, series_diverged,  # noqa: E402
                    series_solve_adaptive)
from oracle.dense import dense_ZF, dense_ZN, direct_solve   # noqa: E402
from hmgen.build import read_rhs                             # noqa: E402
from paper_2109_04129_b200 import PsError                   # noqa: E402
from paper_2109_04129_b200.binding import PS_EDIVERGED, PS_EINVAL  # noqa: E402
from tests.conftest import rel_l2_cols                      # noqa: E402
from tests.test_gpu_parity import _load                     # noqa: E402  (shared handle / oracle cache)

pytestmark = pytest.mark.gpu
TOL = 1e-11


def _dev(A):
    A = np.asfortranarray(A, dtype=np.complex128)
    return torch.from_numpy(np.ascontiguousarray(A.T)).cuda().T


def _host(T):
    return np.asfortranarray(T.T.cpu().numpy().T)


def _oracle(H, S, B, max_terms, tol):
    b_o = apply_Dinv(S, apply_Rt(S, B[S.e2rwg]))
    xt, norms, psum, nt = series_solve_adaptive(lambda v: apply_U(H, S, v), b_o, max_terms, tol)
    x = np.empty_like(xt)
    x[S.e2rwg] = apply_R(S, xt)
    return x, np.array(norms), np.array(psum), nt


def _check(path, B, max_terms, tol=0.0):
    H, S, h = _load(path)
    x_ref, norms, psum, nt = _oracle(H, S, B, max_terms, tol)
    Bd = _dev(B)
    Xd = torch.empty_like(Bd)
    st, rep = h.solve_series(Bd, Xd, max_terms=max_terms, tol=tol)
    if tol > 0 and rep["n_terms"] != nt:
        # the stop is a floating-point comparison on both sides: differ only at a near tie
        n = min(nt, rep["n_terms"]) - 1
        margin = np.abs(norms[n] - tol * psum[n]) / (tol * psum[n])
        assert margin.min() < 1e-9, (rep["n_terms"], nt)
        pytest.skip("stopping decision at a floating-point tie")
    assert rep["n_terms"] == nt
    x = _host(Xd)
    err = rel_l2_cols(x, x_ref)
    assert err.max() <= TOL, err.max()
    assert np.allclose(rep["it_norm"], norms, rtol=1e-10, atol=0)
    div = series_diverged(list(norms))
    assert rep["n_diverged"] == int(div.sum())
    assert (st == PS_EDIVERGED) == bool(div.any())
    X2 = torch.empty_like(Bd)
    h.solve_series(Bd, X2, max_terms=max_terms, tol=tol)
    assert torch.equal(X2, Xd)                     # deterministic
    return x, rep


@pytest.mark.parametrize("n", [1, 2, 3, 7])
def test_series_fixed_terms_synthetic(synthfile, n):
    p, _ = synthfile(n_points=700, seed=4)
    N = _load(p)[2].N
    _check(p, random_rhs(N, 3, seed=n), n)


def test_series_adaptive_reaches_dense_solve(synthfile):
    p, _ = synthfile(n_points=300, seed=8, far_scale=0.05)
    H, S, h = _load(p)
    B = random_rhs(H.N, 2, seed=6)
    x, rep = _check(p, B, 80, 1e-13)
    assert 2 < rep["n_terms"] < 80
    xd = direct_solve(dense_ZN(H) + dense_ZF(H), B)
    assert rel_l2_cols(x, xd).max() < 1e-10


def test_series_ragged_leaves(synthfile):
    p, _ = synthfile(n_points=500, seed=3, clustered=True)
    N = _load(p)[2].N
    for nrhs in (1, 9):
        _check(p, random_rhs(N, nrhs, seed=nrhs), 4)
        _check(p, random_rhs(N, nrhs, seed=nrhs + 1), 30, 1e-9)


def test_series_c1_two_terms_is_ps_solve(cfgdata):
    meta = cfgdata("C1")
    H, S, h = _load(meta["hm"])
    B = random_rhs(H.N, 5, seed=3)
    x2, rep = _check(meta["hm"], B, 2)
    Bd = _dev(B)
    Xd = torch.empty_like(Bd)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _, r2 = h.solve(Bd, Xd)
    assert rel_l2_cols(x2, _host(Xd)).max() <= 1e-12
    assert np.allclose(rep["it_norm"][0], r2["it0"], rtol=1e-12)
    assert np.allclose(rep["it_norm"][1], r2["it1"], rtol=1e-11)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _check(meta["hm"], B, 4)
    # host buffers: the same kernels, bitwise
    Xh = np.zeros_like(np.asfortranarray(B))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h.solve_series(np.asfortranarray(B), Xh, max_terms=4)
        Xd4 = torch.empty_like(Bd)
        h.solve_series(Bd, Xd4, max_terms=4)
    assert np.array_equal(Xh, _host(Xd4))


def test_series_bad_options(synthfile):
    p, _ = synthfile(n_points=700, seed=4)
    h = _load(p)[2]
    B = _dev(random_rhs(h.N, 1, seed=0))
    X = torch.empty_like(B)
    for kw in (dict(max_terms=0), dict(max_terms=5000), dict(max_terms=3, tol=-1.0)):
        with pytest.raises(PsError) as e:
            h.solve_series(B, X, **kw)
        assert e.value.status == PS_EINVAL


@pytest.mark.slow
def test_series_c4_far1p(cfgdata):
    """BASELINE config 3 at 1 and 2 RHS: the narrow plan, whose Z_F is the one-pass far apply
    (far1p), three terms per column."""
    meta = cfgdata("C4")
    B, _ = read_rhs(meta["rhs"])
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _check(meta["hm"], np.asfortranarray(B[:, [0]]), 3)
        _check(meta["hm"], np.asfortranarray(B[:, [90, 270]]), 3)
