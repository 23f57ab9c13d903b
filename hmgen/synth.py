"""Seeded synthetic H-matrices with the structure of the EFIE ones (INPUT GENERATOR).

Random centroids in a box -> the same octree / near list / far interaction
lists / nested-dissection order as the EFIE generator (hmgen.build), but with
random complex-symmetric near blocks and random low-rank far factors. Used by
parity tests to cover structure the physical configs do not hit (size-1 leaves,
ragged sizes, empty far field, a single leaf, controllable ||U||).

Value recipe: near off-diagonal entries ~ CN(0,1)/sqrt(n);
diagonal blocks (A + A^T)/2 + shift * I with shift = diag_shift * (1+1j);
far factors U, V ~ CN(0,1) * far_scale / sqrt(m n)^{1/2}.
"""
from __future__ import annotations

import numpy as np

from .build import HData, build_tree, nd_order


def _cn(rng, *shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2.0)


def synthetic(n_points: int = 400, box: float = 1.0, leaf_edge: float = 0.25, seed: int = 0,
              rank: int = 3, far_scale: float = 0.05, diag_shift: float = 4.0,
              clustered: bool = False) -> HData:
    rng = np.random.default_rng(seed)
    if clustered:
        # a few dense clusters -> very uneven leaf sizes (1 .. many)
        centers = rng.uniform(0, box, size=(6, 3))
        pts = centers[rng.integers(0, 6, n_points)] + 0.08 * box * rng.standard_normal((n_points, 3))
    else:
        pts = rng.uniform(0, box, size=(n_points, 3))
    tree = build_tree(pts, leaf_edge)
    elim = nd_order(tree.leaf_ijk)
    sz = np.diff(tree.leaf_off)
    near_blocks = []
    offs = [0]
    for i, j in tree.near:
        ni, nj = int(sz[i]), int(sz[j])
        if i == j:
            A = _cn(rng, ni, ni)
            Z = 0.5 * (A + A.T) + diag_shift * (1 + 1j) * np.eye(ni)
        else:
            Z = _cn(rng, ni, nj) / np.sqrt(max(ni, nj))
        near_blocks.append(Z)
        offs.append(offs[-1] + ni * nj)
    near_arena = np.concatenate([Z.T.ravel() for Z in near_blocks]) if near_blocks else \
        np.zeros(0, np.complex128)
    near_list = np.stack([tree.near[:, 0], tree.near[:, 1], np.array(offs[:-1])], 1).astype(np.int64)
    far_parts = []
    foffs = [0]
    ranks = []
    for r0, m, c0, n, _lev in tree.far:
        r = int(min(rank, m, n))
        sc = far_scale / np.sqrt(np.sqrt(m * n))
        U = _cn(rng, m, r) * sc
        V = _cn(rng, n, r) * sc
        far_parts.append(np.concatenate([U.T.ravel(), V.T.ravel()]))
        foffs.append(foffs[-1] + r * (m + n))
        ranks.append(r)
    far_arena = np.concatenate(far_parts) if far_parts else np.zeros(0, np.complex128)
    far_list = np.concatenate([tree.far.reshape(-1, 5), np.array(ranks, dtype=np.int64).reshape(-1, 1),
                               np.array(foffs[:-1], dtype=np.int64).reshape(-1, 1)], 1).astype(np.int64)
    stats = dict(N=int(tree.leaf_off[-1]), n_leaves=len(sz), leaf_max=int(sz.max()),
                 leaf_min=int(sz.min()), n_near=len(tree.near), n_far=len(tree.far))
    return HData(int(tree.leaf_off[-1]), 1.0, 2 * np.pi, tree, elim, near_list,
                 near_arena.astype(np.complex128), far_list, far_arena.astype(np.complex128), stats)


def random_rhs(N: int, nrhs: int, seed: int) -> np.ndarray:
    """Complex standard normal right-hand sides (column-major N x nrhs)."""
    rng = np.random.default_rng(1000 + seed)
    return np.asfortranarray(_cn(rng, N, nrhs))
