"""Oracle: dense materialisation for pins (TEST INFRASTRUCTURE ONLY).

  * Z_N, Z_F as dense N x N matrices in RWG order, straight from the file
    (Eqs. 13-14), independent of the scaling code;
  * the closed form of the two-term result:
        x2 = Z_N^{-1} b - Z_N^{-1} Z_F Z_N^{-1} b
    via LAPACK dense LU — the pin for the whole pipeline;
  * the dense-LU solution of the full system Z x = b (§V.A metric,
    ||SOL_dir - SOL_ps|| / ||SOL_dir||).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .hmfile import HMatrix


def dense_ZN(H: HMatrix) -> np.ndarray:
    N = H.N
    Z = np.zeros((N, N), dtype=np.complex128)
    lo = H.leaf_off
    P = H.perm
    for i, j, B in H.near:
        ri = P[lo[i]:lo[i + 1]]
        cj = P[lo[j]:lo[j + 1]]
        Z[np.ix_(ri, cj)] = B
        Z[np.ix_(cj, ri)] = B.T
    return Z


def dense_ZF(H: HMatrix) -> np.ndarray:
    N = H.N
    Z = np.zeros((N, N), dtype=np.complex128)
    P = H.perm
    for r0, m, c0, n, _lev, U, V in H.far:
        rows = P[r0:r0 + m]
        cols = P[c0:c0 + n]
        blk = U @ V.T
        Z[np.ix_(rows, cols)] += blk
        Z[np.ix_(cols, rows)] += blk.T
    return Z


def closed_form_two_term(ZN: np.ndarray, ZF: np.ndarray, B: np.ndarray) -> np.ndarray:
    lu = sla.lu_factor(ZN)
    y0 = sla.lu_solve(lu, B)
    return y0 - sla.lu_solve(lu, ZF @ y0)


def direct_solve(Z: np.ndarray, B: np.ndarray) -> np.ndarray:
    return sla.lu_solve(sla.lu_factor(Z), B)
