"""Oracle-side reader of the `.hm` H-matrix file (TEST INFRASTRUCTURE ONLY).

Independent of libps's C++ loader (read_file in paper_2109_04129_b200/csrc/ps_host.cpp):
written separately from the layout documented in include/ps.h.

Z = Z_N + Z_F (Eq. 13):
  * near blocks Z_ij, i <= j leaf ids, dense (Eq. 14); symmetric
    storage: Z_ji = Z_ij^T;
  * far blocks ~ U V^T (Eq. 11), each symmetric pair stored once.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np


def _checksum(buf: bytes) -> int:
    b = np.frombuffer(buf, dtype=np.uint8)
    n = b.size
    if n % 8:
        b = np.concatenate([b, np.zeros(8 - n % 8, np.uint8)])
    w = b.view("<u8")
    tot = 0
    with np.errstate(over="ignore"):
        for s in range(0, w.size, 1 << 22):
            i = np.arange(s, min(s + (1 << 22), w.size), dtype=np.uint64)
            tot = (tot + int((w[s:s + (1 << 22)] * (2 * i + 1)).sum(dtype=np.uint64))) % (1 << 64)
    return tot ^ n


@dataclass
class HMatrix:
    N: int
    lam: float
    k: float
    perm: np.ndarray       # Morton position -> RWG index
    leaf_off: np.ndarray   # leaf (Morton id) -> first Morton position
    leaf_ijk: np.ndarray
    elim: np.ndarray       # elimination order: position p -> leaf id
    near: list             # [(i, j, Z_ij)] i <= j, Z_ij dense n_i x n_j
    far: list              # [(row0, m, col0, n, level, U (m x r), V (n x r))] Morton positions

    @property
    def n_leaves(self) -> int:
        return len(self.leaf_off) - 1

    def leaf_size(self, leaf: int) -> int:
        return int(self.leaf_off[leaf + 1] - self.leaf_off[leaf])


def read_hm(path: str, verify: bool = True, mmap: bool = False) -> HMatrix:
    """mmap=True maps the file read-only instead of reading it into memory (large
    configs: the block views then page in on use). The values are the same."""
    if mmap:
        data = np.memmap(path, dtype=np.uint8, mode="r")
    else:
        with open(path, "rb") as f:
            data = f.read()
    o = 0

    def take(nbytes):
        nonlocal o
        b = data[o:o + nbytes]
        o += nbytes
        return b

    hdr = bytes(take(4 + 4 + 5 * 8 + 3 * 8 + 8 + 4 * 8 + 2 * 8))
    if hdr[:4] != b"HMPS":
        raise ValueError("bad magic")
    (ver,) = struct.unpack_from("<I", hdr, 4)
    if ver != 1:
        raise ValueError(f"unsupported version {ver}")
    N, nl, nn, nf, flags = struct.unpack_from("<5q", hdr, 8)
    lam, k, _leaf_edge = struct.unpack_from("<3d", hdr, 48)
    n_near_arena, n_far_arena = struct.unpack_from("<2q", hdr, 112)
    (ck,) = struct.unpack("<Q", bytes(take(8)))
    if verify and ck != _checksum(hdr):
        raise ValueError("header checksum mismatch")

    def section(dtype, count):
        nb = np.dtype(dtype).itemsize * count
        raw = take(nb)
        take((-nb) % 8)
        (c,) = struct.unpack("<Q", bytes(take(8)))
        if verify and c != _checksum(raw):
            raise ValueError("section checksum mismatch")
        return np.frombuffer(raw, dtype=dtype, count=count)

    perm = section("<i8", N)
    leaf_off = section("<i8", nl + 1)
    leaf_ijk = section("<i4", nl * 3).reshape(nl, 3)
    elim = section("<i4", nl)
    near_list = section("<i8", nn * 3).reshape(nn, 3)
    near_arena = section("<c16", n_near_arena)
    far_list = section("<i8", nf * 7).reshape(nf, 7)
    far_arena = section("<c16", n_far_arena)
    sz = np.diff(leaf_off)
    near = []
    for i, j, off in near_list:
        ni, nj = int(sz[i]), int(sz[j])
        Z = near_arena[off:off + ni * nj].reshape(nj, ni).T  # column-major n_i x n_j
        near.append((int(i), int(j), Z))
    far = []
    for r0, m, c0, n, lev, r, off in far_list:
        U = far_arena[off:off + m * r].reshape(r, m).T
        V = far_arena[off + m * r:off + m * r + n * r].reshape(r, n).T
        far.append((int(r0), int(m), int(c0), int(n), int(lev), U, V))
    return HMatrix(int(N), lam, k, perm, leaf_off, leaf_ijk, elim, near, far)
