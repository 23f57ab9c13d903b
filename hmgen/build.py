"""Generator pipeline: geometry -> RWG -> octree -> near/far lists -> ND order
-> EFIE near fill + ACA far fill (C++ via ctypes) -> `.hm` file.

Paper passages followed:
  * RWG + Galerkin, Eq. (9).
  * tree partition / admissibility, Eq. (10), PAPER.md:77-83 — realised as the
    octree of BASELINE.json's configs (leaf edge 0.25 lambda), R13.
  * ACA, Eqs. (11)-(12), with recompression [20,21].
  * leaf elimination order: PAPER.md:171 uses Sloan; we use nested dissection
    on the leaf boxes (R3) and store it in the file.

Everything here is deterministic (no random numbers); the only randomness in
the project (random test RHS) is drawn in hmgen.rhs with explicit seeds.
"""
from __future__ import annotations

import ctypes
import hashlib
import json
import math
import os
import struct
import subprocess
import time
from dataclasses import dataclass, field

import numpy as np

C0 = 3.0e8                      # speed of light used for lambda (BASELINE: 300 MHz -> lambda = 1 m)
ETA0 = 120.0 * math.pi          # free-space impedance consistent with C0
HM_MAGIC = b"HMPS"
HM_VERSION = 1

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libefie.so")


# ---------------------------------------------------------------- C++ library
def build_efie(force: bool = False) -> str:
    src = os.path.join(_HERE, "csrc", "efie.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        cmd = ["g++", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC", "-std=c++17",
               src, "-o", _SO]
        subprocess.check_call(cmd)
    return _SO


class EfieLib:
    """ctypes wrapper of hmgen/csrc/efie.cpp (operator assembly, §II)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            build_efie()
            L = ctypes.CDLL(_SO)
            P = ctypes.c_void_p
            I = ctypes.c_int64
            D = ctypes.c_double
            L.efie_create.restype = P
            L.efie_create.argtypes = [I, P, I, P, I, P, P, P, P, D, D]
            L.efie_destroy.argtypes = [P]
            L.efie_block.argtypes = [P, I, P, I, P, P]
            L.efie_near.argtypes = [P, I, P, P, P, P, P, P, P, P]
            L.efie_far.restype = P
            L.efie_far.argtypes = [P, I, P, P, P, P, P, D, P, P]
            L.efie_far_copy.argtypes = [P, I, P, P]
            L.efie_far_free.argtypes = [P]
            L.efie_potential.argtypes = [P, P, P, P]
            L.efie_rhs.argtypes = [P, I, P, P, P]
            L.efie_farfield.argtypes = [P, P, I, P, P]
            cls._lib = L
        return cls._lib

    def __init__(self, mesh: "Mesh", basis: "Rwg", k: float, eta: float = ETA0):
        L = self.lib()
        self._keep = [np.ascontiguousarray(mesh.nodes, dtype=np.float64),
                      np.ascontiguousarray(mesh.tris, dtype=np.int64),
                      np.ascontiguousarray(basis.tp, dtype=np.int64),
                      np.ascontiguousarray(basis.tm, dtype=np.int64),
                      np.ascontiguousarray(basis.vp, dtype=np.int64),
                      np.ascontiguousarray(basis.vm, dtype=np.int64)]
        nd, tr, tp, tm, vp, vm = self._keep
        self.N = basis.N
        self.k = k
        self.h = L.efie_create(len(nd), nd.ctypes.data, len(tr), tr.ctypes.data, basis.N,
                               tp.ctypes.data, tm.ctypes.data, vp.ctypes.data, vm.ctypes.data,
                               float(k), float(eta))

    def __del__(self):
        if getattr(self, "h", None) and self._lib is not None:
            self._lib.efie_destroy(self.h)
            self.h = None

    def block(self, rows, cols) -> np.ndarray:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.zeros((len(cols), len(rows)), dtype=np.complex128)  # column-major m x n
        self.lib().efie_block(self.h, len(rows), rows.ctypes.data, len(cols), cols.ctypes.data,
                              out.ctypes.data)
        return out.T

    def rhs(self, khat: np.ndarray, epol: np.ndarray) -> np.ndarray:
        khat = np.ascontiguousarray(khat, dtype=np.float64)
        ep = np.ascontiguousarray(epol.astype(np.complex128))
        nrhs = khat.shape[0]
        out = np.zeros((nrhs, self.N), dtype=np.complex128)
        self.lib().efie_rhs(self.h, nrhs, khat.ctypes.data, ep.ctypes.data, out.ctypes.data)
        return np.asfortranarray(out.T)

    def farfield(self, I: np.ndarray, rhat: np.ndarray) -> np.ndarray:
        I = np.ascontiguousarray(I, dtype=np.complex128)
        rhat = np.ascontiguousarray(rhat, dtype=np.float64)
        out = np.zeros((rhat.shape[0], 3), dtype=np.complex128)
        self.lib().efie_farfield(self.h, I.ctypes.data, rhat.shape[0], rhat.ctypes.data,
                                 out.ctypes.data)
        return out


def potential_integrals(tri: np.ndarray, r: np.ndarray):
    """Analytic Int_T 1/R dS' and Int_T (r'-r)/R dS' (exposed for tests)."""
    L = EfieLib.lib()
    tri = np.ascontiguousarray(tri, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    js = np.zeros(1)
    jv = np.zeros(3)
    L.efie_potential(tri.ctypes.data, r.ctypes.data, js.ctypes.data, jv.ctypes.data)
    return js[0], jv


# ---------------------------------------------------------------- geometry
@dataclass
class Mesh:
    nodes: np.ndarray   # (n, 3)
    tris: np.ndarray    # (t, 3) int64


def icosphere(radius: float, subdiv: int) -> Mesh:
    t = (1.0 + 5 ** 0.5) / 2.0
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t],
                  [0, -1, -t], [0, 1, -t], [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]],
                 dtype=np.float64)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9],
                  [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2],
                  [3, 2, 6], [3, 6, 8], [3, 8, 9], [4, 9, 5], [2, 4, 11], [6, 2, 10],
                  [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    for _ in range(subdiv):
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
        e.sort(axis=1)
        ue, inv = np.unique(e, axis=0, return_inverse=True)
        mid = v[ue[:, 0]] + v[ue[:, 1]]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        nv = len(v)
        v = np.concatenate([v, mid])
        nf = len(f)
        a = nv + inv[:nf]
        b = nv + inv[nf:2 * nf]
        c = nv + inv[2 * nf:]
        f = np.concatenate([np.stack([f[:, 0], a, c], 1), np.stack([f[:, 1], b, a], 1),
                            np.stack([f[:, 2], c, b], 1), np.stack([a, b, c], 1)])
    return Mesh(v * radius, f)


def cube_mesh(side: float, div: int) -> Mesh:
    """Closed cube, each face a div x div grid of squares split into 2 triangles."""
    nodes = {}
    coords = []

    def nid(p):
        key = tuple(p)
        if key not in nodes:
            nodes[key] = len(coords)
            coords.append(key)
        return nodes[key]

    tris = []
    for axis in range(3):
        for sgn in (0, div):
            u, w = [a for a in range(3) if a != axis]
            for i in range(div):
                for j in range(div):
                    q = []
                    for di, dj in ((0, 0), (1, 0), (1, 1), (0, 1)):
                        p = [0, 0, 0]
                        p[axis] = sgn
                        p[u] = i + di
                        p[w] = j + dj
                        q.append(nid(p))
                    if sgn == 0:
                        q = q[::-1]
                    tris.append([q[0], q[1], q[2]])
                    tris.append([q[0], q[2], q[3]])
    pts = np.array(coords, dtype=np.float64) * (side / div) - side / 2.0
    return Mesh(pts, np.array(tris, dtype=np.int64))


def cylinder_mesh(radius: float, length: float, h: float) -> Mesh:
    """Closed circular cylinder (axis z) with flat caps, near-equilateral triangles of
    edge ~h: the lateral rings are staggered by half a step (ring spacing h*sqrt(3)/2),
    each cap is concentric rings of spacing h*sqrt(3)/2 and circumferential step ~h,
    zipped ring to ring and fanned to the centre."""
    nphi = max(6, int(round(2 * math.pi * radius / h)))
    nz = max(1, int(round(length / (h * math.sqrt(3) / 2))))
    nr = max(1, int(round(radius / (h * math.sqrt(3) / 2))))
    pts = []
    lat = np.zeros((nz + 1, nphi), dtype=np.int64)
    ring_ang = []
    for iz in range(nz + 1):
        z = -length / 2 + length * iz / nz
        a = 2 * math.pi * (np.arange(nphi) + 0.5 * (iz % 2)) / nphi
        ring_ang.append(a)
        for ip in range(nphi):
            lat[iz, ip] = len(pts)
            pts.append((radius * math.cos(a[ip]), radius * math.sin(a[ip]), z))
    tris = []

    def zipper(A, aa, B, bb, out):
        """Triangulate the band between two closed rings (ids A, B; angles aa, bb)."""
        oa, ob = np.argsort(aa % (2 * math.pi)), np.argsort(bb % (2 * math.pi))
        A, aa = A[oa], aa[oa] % (2 * math.pi)
        B, bb = B[ob], bb[ob] % (2 * math.pi)
        # start both rings at the point closest to angle 0 (deterministic)
        ia = ib = 0
        na, nb = len(A), len(B)
        while ia < na or ib < nb:
            a0, a1 = A[ia % na], A[(ia + 1) % na]
            b0, b1 = B[ib % nb], B[(ib + 1) % nb]
            ta = aa[(ia + 1) % na] + (2 * math.pi if ia + 1 >= na else 0)
            tb = bb[(ib + 1) % nb] + (2 * math.pi if ib + 1 >= nb else 0)
            if ib >= nb or (ia < na and ta <= tb):
                out.append([a0, a1, b0])
                ia += 1
            else:
                out.append([a0, b1, b0])
                ib += 1

    for iz in range(nz):
        band = []
        zipper(lat[iz], ring_ang[iz], lat[iz + 1], ring_ang[iz + 1], band)
        tris.extend(band)

    def cap(rim_ids, rim_ang, z, outward_up):
        rings = [rim_ids]
        angs = [rim_ang]
        for ir in range(nr - 1, 0, -1):
            rr = radius * ir / nr
            n = max(6, int(round(2 * math.pi * rr / h)))
            a = 2 * math.pi * (np.arange(n) + 0.5 * ((nr - ir) % 2)) / n
            ids = []
            for t in a:
                ids.append(len(pts))
                pts.append((rr * math.cos(t), rr * math.sin(t), z))
            rings.append(np.array(ids))
            angs.append(a)
        center = len(pts)
        pts.append((0.0, 0.0, z))
        out = []
        for k in range(len(rings) - 1):
            zipper(rings[k], angs[k], rings[k + 1], angs[k + 1], out)
        last = rings[-1]
        order = np.argsort(angs[-1] % (2 * math.pi))
        last = last[order]
        for i in range(len(last)):
            out.append([last[i], last[(i + 1) % len(last)], center])
        for t in out:
            if not outward_up:
                t = [t[0], t[2], t[1]]
            tris.append(t)

    cap(lat[0], ring_ang[0], -length / 2, False)
    cap(lat[nz], ring_ang[nz], length / 2, True)
    return Mesh(np.array(pts, dtype=np.float64), np.array(tris, dtype=np.int64))


def mean_edge(mesh: Mesh) -> float:
    """Mean length over all (unique) mesh edges."""
    e = np.concatenate([mesh.tris[:, [0, 1]], mesh.tris[:, [1, 2]], mesh.tris[:, [2, 0]]])
    e = np.unique(np.sort(e, axis=1), axis=0)
    return float(np.linalg.norm(mesh.nodes[e[:, 0]] - mesh.nodes[e[:, 1]], axis=1).mean())


def cylinder_mesh_mean_edge(radius: float, length: float, target: float) -> Mesh:
    """cylinder_mesh whose MEASURED mean edge (over all edges) is `target` to within
    ~1 %: two fixed-point rescalings of the lattice step (deterministic)."""
    h = target
    m = cylinder_mesh(radius, length, h)
    for _ in range(2):
        h *= target / mean_edge(m)
        m = cylinder_mesh(radius, length, h)
    return m


@dataclass
class Rwg:
    N: int
    edges: np.ndarray   # (N, 2) node ids, sorted (min, max); basis order = sorted edges
    tp: np.ndarray
    tm: np.ndarray
    vp: np.ndarray
    vm: np.ndarray
    center: np.ndarray  # edge midpoints (clustering centroid, R12)
    length: np.ndarray


def rwg_basis(mesh: Mesh) -> Rwg:
    """One RWG function per interior edge, sorted by (min,max) node."""
    f = mesh.tris
    nt = len(f)
    e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
    opp = np.concatenate([f[:, 2], f[:, 0], f[:, 1]])
    tri = np.concatenate([np.arange(nt)] * 3)
    e = np.sort(e, axis=1)
    order = np.lexsort((tri, e[:, 1], e[:, 0]))
    e, opp, tri = e[order], opp[order], tri[order]
    key = e[:, 0] * (len(mesh.nodes) + 1) + e[:, 1]
    uk, start, cnt = np.unique(key, return_index=True, return_counts=True)
    if np.any(cnt > 2):
        raise ValueError("non-manifold edge")
    interior = cnt == 2
    s = start[interior]
    edges = e[s]
    tp, tm = tri[s], tri[s + 1]
    vp, vm = opp[s], opp[s + 1]
    P = mesh.nodes
    center = 0.5 * (P[edges[:, 0]] + P[edges[:, 1]])
    length = np.linalg.norm(P[edges[:, 0]] - P[edges[:, 1]], axis=1)
    return Rwg(len(edges), edges, tp, tm, vp, vm, center, length)


# ---------------------------------------------------------------- octree
def _part1by2(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64) & np.uint64(0x1FFFFF)
    x = (x | (x << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    x = (x | (x << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    x = (x | (x << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    x = (x | (x << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    x = (x | (x << np.uint64(2))) & np.uint64(0x1249249249249249)
    return x


def morton(ijk: np.ndarray) -> np.ndarray:
    return (_part1by2(ijk[:, 0]) << np.uint64(2)) | (_part1by2(ijk[:, 1]) << np.uint64(1)) | \
        _part1by2(ijk[:, 2])


@dataclass
class Tree:
    L: int
    origin: np.ndarray
    root_edge: float
    leaf_edge: float
    perm: np.ndarray        # Morton position -> RWG index
    leaf_off: np.ndarray    # (nleaf+1,)
    leaf_ijk: np.ndarray    # (nleaf, 3)
    near: np.ndarray        # (nnear, 2) leaf pairs i <= j
    far: np.ndarray         # (nfar, 5): row0, m, col0, n, level  (Morton positions)


def build_tree(centers: np.ndarray, leaf_edge: float) -> Tree:
    """Octree with leaf edge `leaf_edge` (R13)."""
    lo, hi = centers.min(0), centers.max(0)
    extent = float((hi - lo).max())
    L = max(0, int(math.ceil(math.log2(max(extent / leaf_edge, 1.0)))))
    # guarantee every centroid is strictly inside the root cube
    root = leaf_edge * 2 ** L
    if root <= extent * (1 + 1e-12):
        L += 1
        root = leaf_edge * 2 ** L
    origin = 0.5 * (lo + hi) - root / 2
    nb = 2 ** L
    ijk = np.floor((centers - origin) / leaf_edge).astype(np.int64)
    ijk = np.clip(ijk, 0, nb - 1)
    code = morton(ijk)
    perm = np.lexsort((np.arange(len(centers)), code))
    code_s = code[perm]
    ucode, start = np.unique(code_s, return_index=True)
    leaf_off = np.concatenate([start, [len(centers)]]).astype(np.int64)
    leaf_ijk = ijk[perm][start]
    nleaf = len(ucode)
    # near list: Chebyshev distance <= 1 (26 neighbours)
    lut = {tuple(x): i for i, x in enumerate(leaf_ijk.tolist())}
    near = []
    offs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)]
    for i, (x, y, z) in enumerate(leaf_ijk.tolist()):
        for a, b, c in offs:
            j = lut.get((x + a, y + b, z + c))
            if j is not None and j >= i:
                near.append((i, j))
    near = np.array(sorted(near), dtype=np.int64).reshape(-1, 2)
    # far lists: interaction lists at levels 2..L
    far = []
    for lev in range(2, L + 1):
        sh = L - lev
        bijk = leaf_ijk >> sh
        bcode = morton(bijk)
        ub, bstart = np.unique(bcode, return_index=True)
        boxes = bijk[bstart]
        bend = np.concatenate([bstart[1:], [nleaf]])
        row0 = leaf_off[bstart]
        rend = leaf_off[bend]
        blut = {tuple(x): i for i, x in enumerate(boxes.tolist())}
        bl = boxes.tolist()
        for i, (x, y, z) in enumerate(bl):
            px, py, pz = x >> 1, y >> 1, z >> 1
            for a, b, c in offs:
                qx, qy, qz = px + a, py + b, pz + c
                for cx in (0, 1):
                    for cy in (0, 1):
                        for cz in (0, 1):
                            key = (2 * qx + cx, 2 * qy + cy, 2 * qz + cz)
                            j = blut.get(key)
                            if j is None or j <= i:
                                continue
                            if max(abs(key[0] - x), abs(key[1] - y), abs(key[2] - z)) > 1:
                                far.append((row0[i], rend[i] - row0[i], row0[j], rend[j] - row0[j], lev))
    far = np.array(sorted(far), dtype=np.int64).reshape(-1, 5)
    return Tree(L, origin, root, leaf_edge, perm.astype(np.int64), leaf_off, leaf_ijk, near, far)


def nd_order(leaf_ijk: np.ndarray) -> np.ndarray:
    """Nested dissection of the leaf boxes (R3).

    Recursive coordinate bisection: split along the axis of largest extent at
    the median box index; the single layer of boxes at that index separates
    the two halves under 26-adjacency. Order = left, right, separator; sets of
    <= 4 boxes keep Morton order (input order)."""
    out = []

    def rec(ids):
        if len(ids) <= 4:
            out.extend(sorted(ids))
            return
        pts = leaf_ijk[ids]
        ext = pts.max(0) - pts.min(0)
        ax = int(np.argmax(ext))
        cs = np.sort(pts[:, ax])
        m = cs[len(cs) // 2]
        left = [i for i, p in zip(ids, pts) if p[ax] < m]
        right = [i for i, p in zip(ids, pts) if p[ax] > m]
        sep = [i for i, p in zip(ids, pts) if p[ax] == m]
        if left:
            rec(left)
        if right:
            rec(right)
        out.extend(sorted(sep))

    rec(list(range(len(leaf_ijk))))
    assert sorted(out) == list(range(len(leaf_ijk)))
    return np.array(out, dtype=np.int32)


# ---------------------------------------------------------------- configs
@dataclass
class Config:
    name: str
    kind: str            # sphere | cube | cylinder
    params: dict
    freq: float
    leaf_frac: float = 0.25
    aca_eps: float = 1e-3
    rhs: str = "theta181"
    desc: str = ""

    @property
    def lam(self):
        return C0 / self.freq

    @property
    def k(self):
        return 2 * math.pi / self.lam


CONFIGS = {
    # tiny configs for unit tests (not BASELINE configs)
    "T0": Config("T0", "sphere", {"radius": 0.5, "subdiv": 1}, 300e6, rhs="x_minus_z",
                 desc="icosphere sub-1 (N=120), r=0.5 m, 300 MHz"),
    "T1": Config("T1", "sphere", {"radius": 0.5, "subdiv": 2}, 300e6, rhs="x_minus_z",
                 desc="icosphere sub-2 (N=480), r=0.5 m, 300 MHz"),
    "T2": Config("T2", "cube", {"side": 1.0, "div": 8}, 300e6, rhs="theta181",
                 desc="cube 1 m, 8x8 per face (N=1152), 300 MHz"),
    # BASELINE.json configs[0..4]
    "C1": Config("C1", "sphere", {"radius": 0.5, "subdiv": 3}, 300e6, rhs="x_minus_z",
                 desc=("PEC sphere r=0.5 m, 300 MHz, icosphere sub-3 (N=1920), 1 RHS x-pol "
                       "along -z")),
    "C2": Config("C2", "cube", {"side": 3.0, "div": 30}, 300e6, rhs="theta181",
                 desc="PEC cube 3 m, 300 MHz, 30x30 per face (N=16200), 181 monostatic RHS"),
    "C3": Config("C3", "sphere", {"radius": 1.0, "subdiv": 5}, 300e6, rhs="theta181",
                 desc="PEC sphere r=1 m, 300 MHz, icosphere sub-5 (N=30720), 181 RHS"),
    "C4": Config("C4", "cylinder", {"radius": 1.0, "length": 10.0}, 600e6, rhs="phi360",
                 desc="PEC cylinder r=1 m, L=10 m, caps, 600 MHz, lambda/10, 360 RHS"),
    "C5": Config("C5", "sphere", {"radius": 3.0, "subdiv": 7}, 300e6, rhs="theta256",
                 desc="PEC sphere r=3 m, 300 MHz, icosphere sub-7 (N=491520), 256 RHS"),
}


def make_mesh(cfg: Config) -> Mesh:
    if cfg.kind == "sphere":
        return icosphere(cfg.params["radius"], cfg.params["subdiv"])
    if cfg.kind == "cube":
        return cube_mesh(cfg.params["side"], cfg.params["div"])
    if cfg.kind == "cylinder":
        return cylinder_mesh_mean_edge(cfg.params["radius"], cfg.params["length"], cfg.lam / 10)
    raise ValueError(cfg.kind)


def plane_wave_dirs(cfg: Config):
    """Incidence table (R19): returns (angles_deg (nrhs,2), khat, epol)."""
    def sph(th, ph):
        st, ct, sp, cp = np.sin(th), np.cos(th), np.sin(ph), np.cos(ph)
        rh = np.stack([st * cp, st * sp, ct], 1)
        th_h = np.stack([ct * cp, ct * sp, -st], 1)
        ph_h = np.stack([-sp, cp, np.zeros_like(sp)], 1)
        return rh, th_h, ph_h

    if cfg.rhs == "x_minus_z":
        th = np.array([0.0]); ph = np.array([0.0]); pol = np.array([0])
    elif cfg.rhs == "theta181":
        th = np.deg2rad(np.arange(181.0)); ph = np.zeros(181); pol = np.zeros(181, int)
    elif cfg.rhs == "theta256":
        th = np.deg2rad(180.0 * np.arange(256) / 255); ph = np.zeros(256); pol = np.zeros(256, int)
    elif cfg.rhs == "phi360":
        ph = np.deg2rad(np.arange(360.0)); th = np.full(360, np.pi / 2)
        pol = (np.arange(360) >= 180).astype(int)
    else:
        raise ValueError(cfg.rhs)
    rh, th_h, ph_h = sph(th, ph)
    khat = -rh
    epol = np.where(pol[:, None] == 0, th_h, ph_h).astype(np.complex128)
    ang = np.stack([np.rad2deg(th), np.rad2deg(ph)], 1)
    return ang, khat, epol


# ---------------------------------------------------------------- checksum
def checksum64(buf) -> int:
    """Weighted 64-bit word sum of a byte buffer (padded with zeros to 8 B):
    h = (sum_i w_i * (2 i + 1)) mod 2^64  XOR  nbytes.  Same definition in
    libps (C++) and oracle/hmfile.py."""
    b = np.frombuffer(memoryview(buf).cast("B"), dtype=np.uint8)
    nbytes = b.size
    pad = (-nbytes) % 8
    if pad:
        b = np.concatenate([b, np.zeros(pad, np.uint8)])
    w = b.view("<u8")
    h = np.uint64(0)
    CH = 1 << 22
    with np.errstate(over="ignore"):
        for s in range(0, w.size, CH):
            idx = np.arange(s, min(s + CH, w.size), dtype=np.uint64)
            h = h + (w[s:s + CH] * (np.uint64(2) * idx + np.uint64(1))).sum(dtype=np.uint64)
    return int(h) ^ nbytes


# ---------------------------------------------------------------- assembly
@dataclass
class HData:
    N: int
    lam: float
    k: float
    tree: Tree
    elim: np.ndarray
    near_list: np.ndarray     # (nnear, 3): i, j, offset (complex entries)
    near_arena: np.ndarray    # complex128
    far_list: np.ndarray      # (nfar, 7): row0, m, col0, n, level, r, offset
    far_arena: np.ndarray
    stats: dict = field(default_factory=dict)


def assemble(cfg: Config, mesh: Mesh | None = None, verbose: bool = False) -> tuple:
    t0 = time.time()
    mesh = mesh if mesh is not None else make_mesh(cfg)
    basis = rwg_basis(mesh)
    tree = build_tree(basis.center, cfg.leaf_frac * cfg.lam)
    elim = nd_order(tree.leaf_ijk)
    efie = EfieLib(mesh, basis, cfg.k)
    lo = tree.leaf_off
    sz = np.diff(lo)
    # near blocks (i <= j, leaf ids in Morton order), column-major n_i x n_j
    ni = sz[tree.near[:, 0]]
    nj = sz[tree.near[:, 1]]
    noff = np.concatenate([[0], np.cumsum(ni * nj)]).astype(np.int64)
    near_arena = np.zeros(int(noff[-1]), dtype=np.complex128)
    idx = np.ascontiguousarray(tree.perm, dtype=np.int64)
    roff = np.ascontiguousarray(lo[tree.near[:, 0]])
    coff = np.ascontiguousarray(lo[tree.near[:, 1]])
    sym = (tree.near[:, 0] == tree.near[:, 1]).astype(np.int64)
    Lb = EfieLib.lib()
    ni_c, nj_c, no_c = (np.ascontiguousarray(x, dtype=np.int64) for x in (ni, nj, noff[:-1]))
    Lb.efie_near(efie.h, len(tree.near), idx.ctypes.data, roff.ctypes.data, ni_c.ctypes.data,
                 coff.ctypes.data, nj_c.ctypes.data, sym.ctypes.data, no_c.ctypes.data,
                 near_arena.ctypes.data)
    t_near = time.time() - t0
    near_list = np.stack([tree.near[:, 0], tree.near[:, 1], noff[:-1]], 1).astype(np.int64)
    # far blocks
    nf = len(tree.far)
    ranks = np.zeros(nf, dtype=np.int64)
    capped = np.zeros(nf, dtype=np.int64)
    fr0 = np.ascontiguousarray(tree.far[:, 0]); fm = np.ascontiguousarray(tree.far[:, 1])
    fc0 = np.ascontiguousarray(tree.far[:, 2]); fn = np.ascontiguousarray(tree.far[:, 3])
    if nf:
        hh = Lb.efie_far(efie.h, nf, idx.ctypes.data, fr0.ctypes.data, fm.ctypes.data,
                         fc0.ctypes.data, fn.ctypes.data, float(cfg.aca_eps), ranks.ctypes.data,
                         capped.ctypes.data)
        fsz = ranks * (fm + fn)
        foff = np.concatenate([[0], np.cumsum(fsz)]).astype(np.int64)
        far_arena = np.zeros(int(foff[-1]), dtype=np.complex128)
        fo = np.ascontiguousarray(foff[:-1])
        Lb.efie_far_copy(hh, nf, fo.ctypes.data, far_arena.ctypes.data)
        Lb.efie_far_free(hh)
    else:
        foff = np.zeros(1, dtype=np.int64)
        far_arena = np.zeros(0, dtype=np.complex128)
    far_list = np.concatenate([tree.far, ranks[:, None], foff[:-1, None]], 1).astype(np.int64)
    stats = dict(N=basis.N, n_tris=len(mesh.tris), n_leaves=len(sz), L=tree.L,
                 leaf_mean=float(sz.mean()), leaf_max=int(sz.max()), n_near=len(tree.near),
                 near_entries=int(noff[-1]), n_far=nf, far_entries=int(foff[-1]),
                 rank_mean=float(ranks.mean()) if nf else 0.0,
                 rank_max=int(ranks.max()) if nf else 0, n_capped=int(capped.sum()),
                 t_near_s=t_near, t_total_s=time.time() - t0)
    if verbose:
        print(json.dumps(stats))
    hd = HData(basis.N, cfg.lam, cfg.k, tree, elim, near_list, near_arena, far_list, far_arena, stats)
    return hd, mesh, basis, efie


def write_hm(path: str, hd: HData) -> None:
    """Write the versioned H-matrix file (layout documented in include/ps.h)."""
    t = hd.tree
    hdr = HM_MAGIC + struct.pack("<I", HM_VERSION)
    hdr += struct.pack("<5q", hd.N, len(t.leaf_off) - 1, len(hd.near_list), len(hd.far_list), 1)
    hdr += struct.pack("<3d", hd.lam, hd.k, t.leaf_edge)
    hdr += struct.pack("<q", t.L)
    hdr += struct.pack("<4d", float(t.origin[0]), float(t.origin[1]), float(t.origin[2]), t.root_edge)
    hdr += struct.pack("<2q", hd.near_arena.size, hd.far_arena.size)
    sections = [np.ascontiguousarray(t.perm, dtype="<i8"),
                np.ascontiguousarray(t.leaf_off, dtype="<i8"),
                np.ascontiguousarray(t.leaf_ijk, dtype="<i4"),
                np.ascontiguousarray(hd.elim, dtype="<i4"),
                np.ascontiguousarray(hd.near_list, dtype="<i8"),
                np.ascontiguousarray(hd.near_arena, dtype="<c16"),
                np.ascontiguousarray(hd.far_list, dtype="<i8"),
                np.ascontiguousarray(hd.far_arena, dtype="<c16")]
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(hdr)
        f.write(struct.pack("<Q", checksum64(hdr)))
        for s in sections:
            mv = memoryview(s.reshape(-1).view(np.uint8)) if s.size else memoryview(b"")
            f.write(mv)
            pad = (-len(mv)) % 8
            if pad:
                f.write(b"\0" * pad)
            f.write(struct.pack("<Q", checksum64(mv)))
    os.replace(tmp, path)


def write_rhs(path: str, B: np.ndarray, ang: np.ndarray) -> None:
    """RHS file: magic 'PSRH', i64 N, i64 nrhs, angles (nrhs x 2 f64), B column-major c16."""
    B = np.asfortranarray(B, dtype=np.complex128)
    with open(path + ".tmp", "wb") as f:
        f.write(b"PSRH")
        f.write(struct.pack("<I", 1))
        f.write(struct.pack("<2q", B.shape[0], B.shape[1]))
        f.write(np.ascontiguousarray(ang, dtype="<f8").tobytes())
        f.write(B.T.astype("<c16").tobytes())
    os.replace(path + ".tmp", path)


def read_rhs(path: str):
    with open(path, "rb") as f:
        assert f.read(4) == b"PSRH"
        struct.unpack("<I", f.read(4))
        N, nrhs = struct.unpack("<2q", f.read(16))
        ang = np.frombuffer(f.read(16 * nrhs), dtype="<f8").reshape(nrhs, 2)
        B = np.frombuffer(f.read(16 * N * nrhs), dtype="<c16").reshape(nrhs, N).T
    return np.asfortranarray(B), ang


def cache_dir() -> str:
    d = os.environ.get("PS_DATA_DIR", os.path.join(os.path.dirname(_HERE), "data"))
    os.makedirs(d, exist_ok=True)
    return d


def _src_digest() -> str:
    h = hashlib.sha256()
    for p in (os.path.join(_HERE, "csrc", "efie.cpp"), os.path.abspath(__file__)):
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:12]


def generate(name: str, outdir: str | None = None, verbose: bool = True) -> dict:
    """Generate config `name` (.hm + .rhs + .json stats) into outdir."""
    cfg = CONFIGS[name]
    outdir = outdir or cache_dir()
    hd, mesh, basis, efie = assemble(cfg, verbose=verbose)
    hm = os.path.join(outdir, f"{name}.hm")
    rh = os.path.join(outdir, f"{name}.rhs")
    write_hm(hm, hd)
    ang, khat, epol = plane_wave_dirs(cfg)
    B = efie.rhs(khat, epol)
    write_rhs(rh, B, ang)
    np.savez(os.path.join(outdir, f"{name}.mesh.npz"), nodes=mesh.nodes, tris=mesh.tris)
    meta = dict(hd.stats, name=name, desc=cfg.desc, digest=_src_digest(), nrhs=B.shape[1])
    with open(os.path.join(outdir, f"{name}.json"), "w") as f:
        json.dump(meta, f, indent=1)
    return meta


def load_or_generate(name: str, outdir: str | None = None, verbose: bool = False) -> dict:
    """Paths of config `name`, regenerating when missing or stale."""
    outdir = outdir or cache_dir()
    js = os.path.join(outdir, f"{name}.json")
    meta = None
    if os.path.exists(js):
        with open(js) as f:
            meta = json.load(f)
        if meta.get("digest") != _src_digest() or not os.path.exists(os.path.join(outdir, f"{name}.hm")):
            meta = None
    if meta is None:
        meta = generate(name, outdir, verbose=verbose)
    meta = dict(meta, hm=os.path.join(outdir, f"{name}.hm"), rhs=os.path.join(outdir, f"{name}.rhs"),
                mesh=os.path.join(outdir, f"{name}.mesh.npz"))
    return meta


def build_config(name: str) -> dict:
    return load_or_generate(name, verbose=True)


if __name__ == "__main__":
    import sys
    for nm in sys.argv[1:]:
        print(json.dumps(generate(nm)))
