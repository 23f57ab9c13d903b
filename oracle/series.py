"""Oracle: the two-term power-series solve (TEST INFRASTRUCTURE ONLY).

PAPER.md §III, in the paper's order, for a block of right-hand sides (columns):

  Eq. (24), PAPER.md:151  b~ = [alpha'_n]...[alpha'_2][alpha'_1] b, alpha'_k = alpha_k^T
                          (PAPER.md:171).  Eq. (25)'s printed transposes are taken as a
                          typo (R1): b~ = R^T b.
  Eq. (32), PAPER.md:185  b_o = Z~_N^{-1} b~
  Eq. (31), PAPER.md:183  U v = Z~_N^{-1} [alpha'...] Z_F [alpha...] v   (far field only)
  Eqs. (35)-(36), PAPER.md:195-197  x~ = b_o - U b_o  (two terms, R2)
  Eq. (26), PAPER.md:157  x = [alpha_1][alpha_2]...[alpha_n] x~
  Eqs. (44)-(45), PAPER.md:239-245  ratio ||it_1|| / ||it_0|| (2-norm per column),
                          converged iff < 0.1 (R7).

Vectors are N x nrhs arrays in elimination order (leaf position blocks), except
for the public `solve`, which takes and returns RWG-ordered columns.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .hmfile import HMatrix
from .scaling import Scaling


def _blk(S: Scaling, v: np.ndarray, k: int) -> np.ndarray:
    return v[S.offsets[k]:S.offsets[k + 1]]


def apply_Rt(S: Scaling, b: np.ndarray) -> np.ndarray:
    """b~ = alpha'_{n} ... alpha'_1 b: apply alpha'_1 = alpha_1^T first (Eq. 24).
    alpha_k^T acts as: block j += alpha_kj^T block k, for j in struct(k)."""
    y = np.array(b, dtype=np.complex128, copy=True)
    for k in range(S.n):
        yk = _blk(S, y, k).copy()
        for j, a in S.alpha[k].items():
            _blk(S, y, j)[...] += a.T @ yk
    return y


def apply_R(S: Scaling, v: np.ndarray) -> np.ndarray:
    """x = alpha_1 alpha_2 ... alpha_{n} v (Eq. 26): the right-most factor acts
    first, so k runs from the last leaf down; alpha_k acts as
    block k += sum_j alpha_kj block j."""
    y = np.array(v, dtype=np.complex128, copy=True)
    for k in range(S.n - 1, -1, -1):
        acc = _blk(S, y, k).copy()
        for j, a in S.alpha[k].items():
            acc = acc + a @ _blk(S, y, j)
        _blk(S, y, k)[...] = acc
    return y


def apply_Dinv(S: Scaling, v: np.ndarray) -> np.ndarray:
    """Z~_N^{-1} v, block diagonal (Eqs. 23, 30, 32)."""
    y = np.empty_like(np.asarray(v, dtype=np.complex128))
    for k in range(S.n):
        _blk(S, y, k)[...] = S.Dinv[k] @ _blk(S, v, k)
    return y


def apply_ZF(H: HMatrix, S: Scaling, w: np.ndarray) -> np.ndarray:
    """t = Z_F w (Eq. 13 far part; far blocks only, never near).
    Each stored block b (rows t_b, cols s_b) is one symmetric pair:
    t[t_b] += U (V^T w[s_b]) and t[s_b] += V (U^T w[t_b])."""
    wm = np.zeros_like(w)
    wm[S.e2mort] = w                      # elimination order -> Morton order
    tm = np.zeros_like(wm)
    for r0, m, c0, n, _lev, U, V in H.far:
        tm[r0:r0 + m] += U @ (V.T @ wm[c0:c0 + n])
        tm[c0:c0 + n] += V @ (U.T @ wm[r0:r0 + m])
    return tm[S.e2mort]


def apply_U(H: HMatrix, S: Scaling, v: np.ndarray) -> np.ndarray:
    """U v = Z~_N^{-1} R^T Z_F R v (Eq. 31)."""
    return apply_Dinv(S, apply_Rt(S, apply_ZF(H, S, apply_R(S, v))))


def check_convergence(ratios, threshold: float = 0.1) -> str:
    """Eq. (45) / PAPER.md:245: ok iff every ratio < threshold."""
    return "ok" if all(float(r) < threshold for r in np.atleast_1d(ratios)) else "diverged"


def series_solve(apply_op, b_o: np.ndarray, n_terms: int = 2):
    """Eq. (36): x~ = sum_{n < n_terms} (-1)^n it_n, it_0 = b_o, it_n = U it_{n-1}.
    Returns x~ and the per-term column norms ||it_n|| (Eq. 44)."""
    it = np.array(b_o, dtype=np.complex128, copy=True)
    xt = it.copy()
    norms = [np.linalg.norm(it, axis=0)]
    for n in range(1, n_terms):
        it = apply_op(it)
        norms.append(np.linalg.norm(it, axis=0))
        xt = xt + (-1) ** n * it
    return xt, norms


def series_solve_adaptive(apply_op, b_o: np.ndarray, max_terms: int, tol: float):
    """Eq. (36) with the term count chosen as DESIGN.md R25 reads Eqs. (44)-(45): add
    it_n = U it_{n-1} (n = 1, 2, ...) to x~ until n + 1 == max_terms or (tol > 0 and
    n >= 1 and every column has ||it_n|| <= tol ||x~_{n+1}||, x~_{n+1} = the partial sum
    through it_n). Returns x~, the per-term norms ||it_n||, the partial-sum norms
    ||x~_{n+1}|| and the number of terms summed."""
    it = np.array(b_o, dtype=np.complex128, copy=True)
    xt = it.copy()
    norms = [np.linalg.norm(it, axis=0)]
    psum = [np.linalg.norm(xt, axis=0)]
    n = 0
    for n in range(1, max_terms):
        it = apply_op(it)
        xt = xt + (-1) ** n * it
        norms.append(np.linalg.norm(it, axis=0))
        psum.append(np.linalg.norm(xt, axis=0))
        if tol > 0 and np.all(norms[-1] <= tol * psum[-1]):
            break
    return xt, norms, psum, len(norms)


def series_diverged(norms) -> np.ndarray:
    """Per column: the last ratio ||it_n|| / ||it_{n-1}|| (Eq. 45) is >= 1, i.e. the
    terms do not shrink and ||U|| <= 1 fails (R25)."""
    if len(norms) < 2:
        return np.zeros(np.shape(norms[0]), dtype=bool)
    a, b = norms[-2], norms[-1]
    return (a > 0) & ~(b < a)


@dataclass
class SolveResult:
    x: np.ndarray          # N x nrhs, RWG order
    b_tilde: np.ndarray    # intermediates, elimination order
    b_o: np.ndarray
    w: np.ndarray
    t: np.ndarray
    u: np.ndarray
    x_tilde: np.ndarray
    it0: np.ndarray        # ||b_o|| per column
    it1: np.ndarray        # ||U b_o|| per column
    ratio: np.ndarray
    status: str


def solve(H: HMatrix, S: Scaling, B: np.ndarray, threshold: float = 0.1) -> SolveResult:
    """Two-term solve of Z x = b (Eq. 9) for RWG-ordered columns B (N x nrhs)."""
    B = np.asarray(B, dtype=np.complex128)
    squeeze = B.ndim == 1
    if squeeze:
        B = B[:, None]
    b = B[S.e2rwg]                                   # RWG -> elimination order
    b_tilde = apply_Rt(S, b)                         # Eq. (24)
    b_o = apply_Dinv(S, b_tilde)                     # Eq. (32)
    w = apply_R(S, b_o)
    t = apply_ZF(H, S, w)
    u = apply_Dinv(S, apply_Rt(S, t))                # U b_o, Eq. (31)
    x_tilde = b_o - u                                # Eq. (36), two terms
    x_e = apply_R(S, x_tilde)                        # Eq. (26)
    x = np.empty_like(x_e)
    x[S.e2rwg] = x_e
    it0 = np.linalg.norm(b_o, axis=0)
    it1 = np.linalg.norm(u, axis=0)
    ratio = it1 / np.where(it0 > 0, it0, 1.0)
    status = check_convergence(ratio, threshold)
    if squeeze:
        x = x[:, 0]
    return SolveResult(x, b_tilde, b_o, w, t, u, x_tilde, it0, it1, ratio, status)
