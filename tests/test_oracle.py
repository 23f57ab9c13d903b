"""Pins of the ORACLE against what the paper and the mathematics fix (CPU only).

Each pin is chosen so that a plausible mistake (a dropped term, a wrong sign or
index, a transposed operand, a wrong product order) fails at least one:
  * textbook 2-leaf Schur complement (Eq. 21 / SPEC S:413);
  * exact block-diagonalisation R^T Z_N R = diag(D_k) (Eq. 23) on the Eq. (14)
    4-leaf pattern, on random octree systems and on BASELINE config 0;
  * left scaling = transpose of right, bilinear adjoint identity;
  * closed form x2 = Z_N^-1 b - Z_N^-1 Z_F Z_N^-1 b against dense LU;
  * residual pins Z_N w = b and Z_N R u = Z_F w (matrix-free, any size);
  * scalar surrogate U = cI truncation law (Eq. 35);
  * many-term limit = dense solve of Z (Eqs. 33-35); order invariance of x;
  * the literal Eq. (25) reading fails (R1) while Eq. (24)'s holds.
"""
import numpy as np
import pytest

from hmgen.build import read_rhs, write_hm
from hmgen.synth import random_rhs, synthetic
from oracle import (apply_Dinv, apply_R, apply_Rt, apply_U, apply_ZF, check_convergence,
                    compute_scaling, read_hm, series_solve, solve)
from oracle.dense import closed_form_two_term, dense_ZF, dense_ZN, direct_solve
from oracle.hmfile import HMatrix
from oracle.scaling import SingularBlock, dense_R
from tests.conftest import rel_l2_cols


def _cn(rng, *s):
    return rng.standard_normal(s) + 1j * rng.standard_normal(s)


def _hm_from_blocks(sizes, blocks, order=None, far=()):
    """In-memory HMatrix from leaf sizes and {(i,j): Z_ij} (i <= j)."""
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    N = int(off[-1])
    near = [(i, j, Z) for (i, j), Z in sorted(blocks.items())]
    n = len(sizes)
    return HMatrix(N, 1.0, 2 * np.pi, np.arange(N), off, np.zeros((n, 3), np.int32),
                   np.arange(n) if order is None else np.asarray(order), near, list(far))


def test_two_leaf_textbook_schur():
    rng = np.random.default_rng(0)
    A = _cn(rng, 3, 3); A = A + A.T + 8 * np.eye(3)
    C = _cn(rng, 4, 4); C = C + C.T + 8 * np.eye(4)
    B = _cn(rng, 3, 4)
    S = compute_scaling(_hm_from_blocks([3, 4], {(0, 0): A, (0, 1): B, (1, 1): C}))
    assert np.allclose(S.alpha[0][1], -np.linalg.solve(A, B), atol=1e-13)
    assert np.allclose(S.D[0], A)
    assert np.allclose(S.D[1], C - B.T @ np.linalg.solve(A, B), atol=1e-12)
    assert S.alpha[1] == {}                       # the last leaf has no scaling


def test_identity_near_field():
    S = compute_scaling(_hm_from_blocks([2, 3, 1], {(0, 0): np.eye(2), (1, 1): np.eye(3),
                                                    (2, 2): np.eye(1), (0, 1): np.zeros((2, 3))}))
    for k in range(3):
        assert np.allclose(S.Dinv[k], np.eye(S.sizes[k]))
        for a in S.alpha[k].values():
            assert np.allclose(a, 0)


def _eq14_system(seed=1, n=(3, 2, 4, 3)):
    """The 4-leaf near field of Eq. (14): Z_14 = Z_41 = 0, all other pairs coupled."""
    rng = np.random.default_rng(seed)
    blocks = {}
    for i in range(4):
        for j in range(i, 4):
            if (i, j) == (0, 3):
                continue
            Z = _cn(rng, n[i], n[j])
            if i == j:
                Z = Z + Z.T + 10 * np.eye(n[i])
            blocks[(i, j)] = Z
    return _hm_from_blocks(list(n), blocks)


def _dense_ZN_e(H, S):
    Z = dense_ZN(H)
    return Z[np.ix_(S.e2rwg, S.e2rwg)]


def test_eq14_exact_diagonalisation_and_fill():
    H = _eq14_system()
    S = compute_scaling(H)
    assert sorted(S.alpha[0]) == [1, 2]             # Eq. (16): alpha_12, alpha_13; no alpha_14
    assert sorted(S.alpha[1]) == [2, 3]
    R = dense_R(S)
    ZN = _dense_ZN_e(H, S)
    Zt = R.T @ ZN @ R                                # Eq. (22)
    o = S.offsets
    off = Zt.copy()
    for k in range(S.n):
        assert np.allclose(Zt[o[k]:o[k + 1], o[k]:o[k + 1]], S.D[k], atol=1e-12 * np.abs(ZN).max())
        off[o[k]:o[k + 1], o[k]:o[k + 1]] = 0
    assert np.linalg.norm(off) <= 1e-12 * np.linalg.norm(ZN)     # Eq. (23)


def test_sweeps_equal_dense_products_and_adjoint():
    hd = synthetic(n_points=300, seed=2)
    H = _hdata_to_hm(hd)
    S = compute_scaling(H)
    R = dense_R(S)
    rng = np.random.default_rng(7)
    v = _cn(rng, S.N, 3)
    w = _cn(rng, S.N, 3)
    assert np.allclose(apply_R(S, w), R @ w, atol=1e-12 * np.abs(R @ w).max())
    assert np.allclose(apply_Rt(S, v), R.T @ v, atol=1e-12 * np.abs(R.T @ v).max())
    # bilinear (not sesquilinear) adjoint: v^T (R w) = (R^T v)^T w  (R11)
    lhs = np.einsum("ic,ic->c", v, apply_R(S, w))
    rhs = np.einsum("ic,ic->c", apply_Rt(S, v), w)
    assert np.allclose(lhs, rhs, rtol=1e-12)
    ZN = _dense_ZN_e(H, S)
    Zt = R.T @ ZN @ R
    D = np.zeros_like(Zt)
    o = S.offsets
    for k in range(S.n):
        D[o[k]:o[k + 1], o[k]:o[k + 1]] = S.D[k]
    assert np.linalg.norm(Zt - D) <= 1e-12 * np.linalg.norm(ZN)
    # D^{-1} really inverts each scaled block
    x = apply_Dinv(S, v)
    assert np.allclose(D @ x, v, atol=1e-12 * np.abs(v).max())


def _hdata_to_hm(hd):
    import os
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "x.hm")
        write_hm(p, hd)
        return read_hm(p)


def test_closed_form_synthetic_convergent():
    hd = synthetic(n_points=400, seed=4, far_scale=0.05)
    H = _hdata_to_hm(hd)
    S = compute_scaling(H)
    B = random_rhs(H.N, 4, seed=0)
    r = solve(H, S, B)
    ZN, ZF = dense_ZN(H), dense_ZF(H)
    x2 = closed_form_two_term(ZN, ZF, B)
    assert rel_l2_cols(r.x, x2).max() < 1e-13
    assert r.status == "ok" and r.ratio.max() < 0.1
    # truncation error is second order in ||Z_N^-1 Z_F||
    xd = direct_solve(ZN + ZF, B)
    err = rel_l2_cols(r.x, xd)
    assert (err < 5 * r.ratio ** 2).all()


@pytest.mark.parametrize("name", ["C1", "T2"])
def test_closed_form_physical(cfgdata, name):
    meta = cfgdata(name)
    H = read_hm(meta["hm"])
    S = compute_scaling(H)
    B, _ = read_rhs(meta["rhs"])
    B = B[:, :3]
    r = solve(H, S, B)
    ZN, ZF = dense_ZN(H), dense_ZF(H)
    assert rel_l2_cols(r.x, closed_form_two_term(ZN, ZF, B)).max() < 1e-12
    # residual pins (matrix-free form holds at any N): Z_N w = b, Z_N R u = Z_F w
    b_e = B[S.e2rwg]
    ZNe = ZN[np.ix_(S.e2rwg, S.e2rwg)]
    assert rel_l2_cols(ZNe @ r.w, b_e).max() < 1e-13
    assert rel_l2_cols(ZNe @ apply_R(S, r.u), r.t).max() < 1e-13
    # Eq. (23) at full size: off-diagonal of R^T Z_N R vanishes (probe form)
    rng = np.random.default_rng(0)
    v = _cn(rng, H.N, 2)
    lhs = apply_Rt(S, ZNe @ apply_R(S, v))
    o = S.offsets
    Dv = np.concatenate([S.D[k] @ v[o[k]:o[k + 1]] for k in range(S.n)])
    assert np.linalg.norm(lhs - Dv) <= 1e-12 * np.linalg.norm(Dv)


def test_order_invariance():
    """x does not depend on the elimination order (App. B); the ratio does."""
    hd = synthetic(n_points=300, seed=6)
    H = _hdata_to_hm(hd)
    B = random_rhs(H.N, 2, seed=1)
    r1 = solve(H, compute_scaling(H), B)
    order = np.random.default_rng(3).permutation(H.n_leaves)
    r2 = solve(H, compute_scaling(H, order), B)
    assert rel_l2_cols(r2.x, r1.x).max() < 1e-12


def test_scalar_surrogate_truncation_law():
    """U = cI: n-term partial sum = (1 - (-c)^n)/(1 + c) b_o; error vs b_o/(1+c)
    is |c|^n / |1 + c| ||b_o|| (Eq. 35, SPEC S:497 / S:701)."""
    rng = np.random.default_rng(0)
    bo = _cn(rng, 50, 2)
    for c in (0.05, 0.3, 0.8, -0.2 + 0.1j):
        for n in (1, 2, 3, 6):
            xt, norms = series_solve(lambda v: c * v, bo, n_terms=n)
            exact = bo / (1 + c)
            err = np.linalg.norm(xt - exact, axis=0) / np.linalg.norm(bo, axis=0)
            assert np.allclose(err, abs(c) ** n / abs(1 + c), rtol=1e-12)
            if n >= 2:
                assert np.allclose(norms[1] / norms[0], abs(c))
    xt, _ = series_solve(lambda v: 0.3 * v, bo, n_terms=2)
    assert np.allclose(xt, 0.7 * bo)


def test_many_terms_converge_to_dense_solve():
    hd = synthetic(n_points=300, seed=8, far_scale=0.05)
    H = _hdata_to_hm(hd)
    S = compute_scaling(H)
    B = random_rhs(H.N, 2, seed=2)
    b_o = apply_Dinv(S, apply_Rt(S, B[S.e2rwg]))
    xt, norms = series_solve(lambda v: apply_U(H, S, v), b_o, n_terms=40)
    x = np.empty_like(xt)
    x[S.e2rwg] = apply_R(S, xt)
    xd = direct_solve(dense_ZN(H) + dense_ZF(H), B)
    assert rel_l2_cols(x, xd).max() < 1e-10


def test_single_leaf_no_far_field():
    rng = np.random.default_rng(9)
    A = _cn(rng, 5, 5); A = A + A.T + 6 * np.eye(5)
    H = _hm_from_blocks([5], {(0, 0): A})
    S = compute_scaling(H)
    b = _cn(rng, 5, 1)
    r = solve(H, S, b)
    assert np.allclose(r.x, np.linalg.solve(A, b), atol=1e-13)
    assert np.allclose(r.u, 0) and r.status == "ok"


def test_zf_apply_matches_dense():
    hd = synthetic(n_points=250, seed=10)
    H = _hdata_to_hm(hd)
    S = compute_scaling(H)
    w = random_rhs(H.N, 2, seed=3)
    t = apply_ZF(H, S, w[S.e2rwg])
    ref = (dense_ZF(H) @ w)[S.e2rwg]
    assert np.allclose(t, ref, atol=1e-13 * np.abs(ref).max())


def test_literal_eq25_reading_is_wrong():
    """DESIGN.md R1: Eq. (25) printed as b~ = [a'_3]^T[a'_2]^T[a'_1]^T b. Taken
    literally (apply alpha_k instead of alpha_k^T) the result is far from the
    closed form, while Eq. (24)'s b~ = R^T b reproduces it."""
    hd = synthetic(n_points=300, seed=4, far_scale=0.05)
    H = _hdata_to_hm(hd)
    S = compute_scaling(H)
    B = random_rhs(H.N, 1, seed=0)
    b = B[S.e2rwg]
    y = b.copy()
    o = S.offsets
    for k in range(S.n):                                    # literal: alpha_1^... applied as alpha
        for j, a in S.alpha[k].items():
            y[o[k]:o[k + 1]] += a @ y[o[j]:o[j + 1]]
    x_lit = apply_R(S, apply_Dinv(S, y))
    x_ok = apply_R(S, apply_Dinv(S, apply_Rt(S, b)))
    ZN = _dense_ZN_e(H, S)
    ref = np.linalg.solve(ZN, b)
    assert rel_l2_cols(x_ok, ref).max() < 1e-12
    assert rel_l2_cols(x_lit, ref).max() > 1e-2


def test_check_convergence_and_divergence_flag():
    assert check_convergence([0.05, 0.04]) == "ok"
    assert check_convergence([0.5]) == "diverged"
    assert check_convergence([0.1]) == "diverged"            # strict < 0.1 (R7)
    # identity-replaced near field => ratio >= 0.1, diverged (SPEC acceptance 4)
    hd = synthetic(n_points=300, seed=11, far_scale=30.0)
    H = _hdata_to_hm(hd)
    r = solve(H, compute_scaling(H), random_rhs(H.N, 1, seed=0))
    assert r.status == "diverged" and r.ratio[0] >= 0.1


def test_singular_block_named():
    H = _hm_from_blocks([2, 2], {(0, 0): np.zeros((2, 2)), (1, 1): np.eye(2)})
    with pytest.raises(SingularBlock) as e:
        compute_scaling(H)
    assert e.value.leaf == 0


def test_hmfile_checksum_detects_corruption(tmp_path):
    hd = synthetic(n_points=120, seed=12)
    p = str(tmp_path / "c.hm")
    write_hm(p, hd)
    read_hm(p)
    raw = bytearray(open(p, "rb").read())
    raw[len(raw) // 2] ^= 0x40
    q = str(tmp_path / "d.hm")
    open(q, "wb").write(bytes(raw))
    with pytest.raises(ValueError):
        read_hm(q)


def test_spill_and_mmap_storage_are_value_identical(cfgdata, tmp_path):
    """The large-config storage options (memory-mapped file read, alpha blocks spilled to
    a memory-mapped file; used for C5's golden) hold exactly the in-memory values."""
    from oracle import compute_scaling, read_hm, solve
    meta = cfgdata("C1")
    H0 = read_hm(meta["hm"])
    H1 = read_hm(meta["hm"], mmap=True)
    assert all(np.array_equal(a[2], b[2]) for a, b in zip(H0.near, H1.near))
    assert all(np.array_equal(a[5], b[5]) and np.array_equal(a[6], b[6]) for a, b in zip(H0.far, H1.far))
    S0 = compute_scaling(H0)
    S1 = compute_scaling(H1, spill=str(tmp_path / "alpha.bin"))
    for k in range(S0.n):
        assert list(S0.alpha[k]) == list(S1.alpha[k])
        for j in S0.alpha[k]:
            assert np.array_equal(S0.alpha[k][j], S1.alpha[k][j])
    B, _ = read_rhs(meta["rhs"])
    assert np.array_equal(solve(H0, S0, B).x, solve(H1, S1, B).x)


def test_truncation_size_report_c1(cfgdata):
    """SURVEY §8(c) 'truncation size: reported number' (PAPER.md:313 metric): the committed
    tests/golden/accuracy.json (scripts/accuracy_report.py: oracle two-term x vs dense LU of
    Z = Z_N + Z_F) reproduces on C1, and the error is of the size the Eq. 45 ratio implies
    for a two-term truncation (ratio 0.80 >= 0.1: the paper's divergence regime, R14)."""
    import json
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    from accuracy_report import report
    cfgdata("C1")
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "accuracy.json")) as f:
        stored = json.load(f)["C1"]
    now = report("C1")
    e0 = stored["rel_err_two_term_vs_dense_LU"]["max"]
    assert abs(now["rel_err_two_term_vs_dense_LU"]["max"] - e0) <= 1e-10 * e0
    assert abs(now["ratio_it1_it0"]["max"] - stored["ratio_it1_it0"]["max"]) <= 1e-12
    assert 0.1 <= e0 <= 1.0 and now["ratio_it1_it0"]["max"] >= 0.1


# ---- n-term / adaptive series (R25) ----

def test_n_term_series_matches_dense_closed_form():
    """x_n = R sum_{k<n} (-U)^k b_o equals sum_{k<n} (-Z_N^{-1} Z_F)^k Z_N^{-1} b, because
    R U R^{-1} = R D^{-1} R^T Z_F = Z_N^{-1} Z_F (Eqs. 26, 28, 31, 35): dense LU of the
    file's near field, no scaling code on this side."""
    from oracle import series_solve
    hd = synthetic(n_points=260, seed=11, far_scale=0.2)
    H = _hdata_to_hm(hd)
    S = compute_scaling(H)
    B = random_rhs(H.N, 2, seed=4)
    ZN, ZF = dense_ZN(H), dense_ZF(H)
    y = direct_solve(ZN, B)
    ref = np.zeros_like(y)
    term = y.copy()
    b_o = apply_Dinv(S, apply_Rt(S, B[S.e2rwg]))
    for n in range(1, 6):
        ref = ref + term                             # sum_{k<n} (-ZN^-1 ZF)^k ZN^-1 b
        xt, _ = series_solve(lambda v: apply_U(H, S, v), b_o, n_terms=n)
        x = np.empty_like(xt)
        x[S.e2rwg] = apply_R(S, xt)
        assert rel_l2_cols(x, ref).max() < 1e-11, n
        term = -direct_solve(ZN, ZF @ term)


def test_adaptive_series_scalar_surrogate():
    """U = cI: term n has norm |c|^n ||b_o||, the partial sum through it_n is
    (1 - (-c)^{n+1}) / (1 + c) b_o; the rule stops at the first n >= 1 with
    |c|^n <= tol |1 - (-c)^{n+1}| / |1 + c| (R25), else at max_terms."""
    from oracle import series_diverged, series_solve_adaptive
    rng = np.random.default_rng(5)
    bo = _cn(rng, 40, 3)
    for c in (0.05, 0.3, -0.45 + 0.2j, 0.8):
        for tol in (1e-3, 1e-8, 1e-12):
            n_exp = 60
            for n in range(1, 60):
                if abs(c) ** n <= tol * abs(1 - (-c) ** (n + 1)) / abs(1 + c):
                    n_exp = n + 1
                    break
            xt, norms, psum, nt = series_solve_adaptive(lambda v: c * v, bo, 60, tol)
            assert nt == n_exp, (c, tol)
            assert np.allclose(xt, (1 - (-c) ** nt) / (1 + c) * bo, rtol=1e-12, atol=1e-14)
            assert np.allclose(norms[-1], abs(c) ** (nt - 1) * np.linalg.norm(bo, axis=0), rtol=1e-10)
            assert not series_diverged(norms).any()
    # tol = 0: exactly max_terms terms, the same sum as the fixed-n series
    from oracle import series_solve
    xt, norms, _, nt = series_solve_adaptive(lambda v: 0.3 * v, bo, 5, 0.0)
    x5, _ = series_solve(lambda v: 0.3 * v, bo, n_terms=5)
    assert nt == 5 and np.array_equal(xt, x5)
    # |c| >= 1: the terms do not shrink -> diverged
    _, norms, _, nt = series_solve_adaptive(lambda v: -1.2 * v, bo, 4, 1e-6)
    assert nt == 4 and series_diverged(norms).all()


def test_adaptive_series_reaches_dense_solve():
    """On a convergent synthetic system the adaptive series at tol 1e-13 ends within
    1e-10 of the dense-LU solution of Z = Z_N + Z_F (PAPER.md:313 metric), and the
    Eq. 45 ratios settle below 1."""
    from oracle import series_diverged, series_solve_adaptive
    hd = synthetic(n_points=300, seed=8, far_scale=0.05)
    H = _hdata_to_hm(hd)
    S = compute_scaling(H)
    B = random_rhs(H.N, 2, seed=6)
    b_o = apply_Dinv(S, apply_Rt(S, B[S.e2rwg]))
    xt, norms, psum, nt = series_solve_adaptive(lambda v: apply_U(H, S, v), b_o, 80, 1e-13)
    assert 2 < nt < 80
    x = np.empty_like(xt)
    x[S.e2rwg] = apply_R(S, xt)
    xd = direct_solve(dense_ZN(H) + dense_ZF(H), B)
    assert rel_l2_cols(x, xd).max() < 1e-10
    assert not series_diverged(norms).any()
