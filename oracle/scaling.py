"""Oracle: Schur-complement scaling of the symmetric near field (TEST INFRASTRUCTURE ONLY).

Follows PAPER.md §III.A step by step, in the paper's order:

  Eq. (16), PAPER.md:123   alpha_kj = -Z~_kk^{-1} Z~_kj            (right scaling)
  Eq. (18), PAPER.md:129   alpha'_jk = -Z~_jk Z~_kk^{-1} = alpha_kj^T (left; symmetric
                           case: "mere transpose", PAPER.md:171 — never stored)
  Eq. (21), PAPER.md:141   Z~_ij <- Z~_ij - Z~_ik Z~_kk^{-1} Z~_kj = Z~_ij + alpha_ki^T Z~_kj
                           for every pair i, j coupled to k, fill-in included
                           ("considering fill-in blocks")
  Eqs. (22)-(23), PAPER.md:145-147  repeated for every leaf k in elimination order
                           -> block-diagonal Z~_N = diag(Z~_kk); D_k^{-1} = Z~_kk^{-1}.

The elimination order is the file's (nested dissection, R3, in place
of Sloan's ordering of PAPER.md:171). Leaves are addressed by their position
k = 0..n_l-1 in that order. Fill is discovered as the elimination proceeds:
the blocks present in row k when k is eliminated are exactly struct(k).

D_k^{-1}: LU with partial pivoting (LAPACK getrf) followed by inversion
(R5). Singular if a pivot |u_ii| <= 1e-14 ||Z~_kk||_F (R5).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla

from .hmfile import HMatrix


class SingularBlock(ArithmeticError):
    def __init__(self, pos: int, leaf: int):
        super().__init__(f"singular scaled diagonal block at elimination position {pos} (leaf {leaf})")
        self.pos = pos
        self.leaf = leaf


@dataclass
class Scaling:
    n: int                   # number of leaves
    sizes: np.ndarray        # n_k by position
    offsets: np.ndarray      # first unknown of position k in elimination-ordered vectors
    leaf_of: np.ndarray      # position -> leaf id
    alpha: list              # alpha[k] = {j: alpha_kj (n_k x n_j)}, j > k
    Dinv: list               # Dinv[k] = Z~_kk^{-1}
    D: list                  # D[k] = Z~_kk (final scaled diagonal block)
    e2rwg: np.ndarray        # elimination-ordered unknown -> RWG index
    e2mort: np.ndarray       # elimination-ordered unknown -> Morton position

    @property
    def N(self) -> int:
        return int(self.offsets[-1])

    def struct(self, k: int) -> list:
        return sorted(self.alpha[k].keys())


def inverse_lu(A: np.ndarray, pos: int = -1, leaf: int = -1) -> np.ndarray:
    """Explicit inverse via LU with partial pivoting (getrf) + solve with I."""
    lu, piv = sla.lu_factor(A, check_finite=True)
    fro = np.linalg.norm(A)
    if not np.min(np.abs(np.diag(lu))) > 1e-14 * fro:
        raise SingularBlock(pos, leaf)
    return sla.lu_solve((lu, piv), np.eye(A.shape[0], dtype=A.dtype))


class _Spill:
    """Append-only file of finished alpha blocks (large configs whose alpha panels exceed
    host memory): a block is written once its row is scaled out and read back through a
    read-only memory map. Storage only; the values are the same."""

    def __init__(self, path: str):
        self.path = path
        self.f = open(path, "wb")
        self.off = 0
        self.index = []                         # (k, j, offset, n_k, n_j)

    def put(self, k: int, j: int, a: np.ndarray) -> None:
        a = np.ascontiguousarray(a, dtype=np.complex128)
        self.f.write(a.tobytes())
        self.index.append((k, j, self.off, a.shape[0], a.shape[1]))
        self.off += a.size

    def close(self, alpha: list) -> None:
        self.f.close()
        mm = np.memmap(self.path, dtype=np.complex128, mode="r", shape=(max(self.off, 1),))
        for k, j, off, m, n in self.index:
            alpha[k][j] = mm[off:off + m * n].reshape(m, n)


def compute_scaling(H: HMatrix, order: np.ndarray | None = None, spill: str | None = None) -> Scaling:
    """Eqs. (14)-(23) with exact fill-in. `order` overrides the file's elimination order.
    spill: file name; finished alpha blocks are kept there (memory-mapped) instead of in
    memory (C5: 67 GB of panels)."""
    order = np.asarray(H.elim if order is None else order, dtype=np.int64)
    n = len(order)
    pos_of = np.empty(n, dtype=np.int64)
    pos_of[order] = np.arange(n)
    sizes = np.array([H.leaf_size(int(l)) for l in order], dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)

    # Z~ starts as Z_N (Eq. 14): upper blocks (p <= q) by elimination position.
    Zt = {}
    rows = [set() for _ in range(n)]
    for i, j, Z in H.near:
        p, q = int(pos_of[i]), int(pos_of[j])
        blk = np.array(Z, dtype=np.complex128)
        if p <= q:
            Zt[(p, q)] = blk
        else:
            Zt[(q, p)] = blk.T.copy()
        a, b = min(p, q), max(p, q)
        if a != b:
            rows[a].add(b)

    alpha = [dict() for _ in range(n)]
    sp = _Spill(spill) if spill else None
    Dinv = [None] * n
    D = [None] * n
    for k in range(n):
        Zkk = Zt[(k, k)]
        # lower triangle of Z~ is implicit: Z~_kk is symmetric by construction
        D[k] = Zkk
        Dinv[k] = inverse_lu(Zkk, k, int(order[k]))
        row = sorted(rows[k])                 # struct(k), including fill-in
        for j in row:                         # Eq. (16)
            alpha[k][j] = -Dinv[k] @ Zt[(k, j)]
        for a, i in enumerate(row):           # Eq. (21), i <= j
            for j in row[a:]:
                upd = alpha[k][i].T @ Zt[(k, j)]
                if (i, j) in Zt:
                    Zt[(i, j)] = Zt[(i, j)] + upd
                else:
                    Zt[(i, j)] = upd          # fill-in block
                    if i != j:
                        rows[i].add(j)
        # row k is now scaled out (Eq. 21 first row/column = 0); drop it
        for j in row:
            del Zt[(k, j)]
        if sp is not None:
            for j in row:
                sp.put(k, j, alpha[k][j])
            alpha[k] = {j: None for j in row}
    if sp is not None:
        sp.close(alpha)

    # unknown maps: elimination-ordered unknown -> Morton position -> RWG index
    e2mort = np.concatenate([np.arange(H.leaf_off[l], H.leaf_off[l + 1]) for l in order]).astype(np.int64)
    e2rwg = H.perm[e2mort].astype(np.int64)
    return Scaling(n, sizes, offsets, order, alpha, Dinv, D, e2rwg, e2mort)


def dense_R(S: Scaling) -> np.ndarray:
    """Materialise R = alpha_1 alpha_2 ... alpha_{n-1} (Eq. 26) in elimination
    order, column by column, as the product of the elementary matrices of
    Eq. (15) — used only by small pins."""
    N = S.N
    R = np.eye(N, dtype=np.complex128)
    o = S.offsets
    for k in range(S.n):          # R <- R alpha_k  (right-multiplication, Eq. 26 order)
        if not S.alpha[k]:
            continue
        Ak = np.eye(N, dtype=np.complex128)
        for j, a in S.alpha[k].items():
            Ak[o[k]:o[k + 1], o[j]:o[j + 1]] = a
        R = R @ Ak
    return R
