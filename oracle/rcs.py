"""Oracle: far field and RCS of RWG surface currents (TEST INFRASTRUCTURE ONLY).

SURVEY §8(f) NEXT-4, the post-processing after the solve: the bistatic / monostatic RCS
curves of PAPER.md:333-341 (sphere vs Mie), 365, 383-397. Written from the definitions:

  RWG basis (Rao-Wilton-Glisson): f_n(r) = +l_n / (2 A+) (r - v+) on T+,
      -l_n / (2 A-) (r - v-) on T-, l_n the length of the shared edge.
  Far-field vector of the currents x (Eq. 9's unknowns):
      F(r^) = sum_n x_n int_{T+ u T-} f_n(r') exp(+j k r^ . r') dS'
  (e^{+jwt}, G = e^{-jkR}/(4 pi R), R16: the far-zone G is e^{-jkr}/(4 pi r)
  e^{+jk r^.r'}), each triangle integral by the 7-point degree-5 rule (Dunavant 1985;
  DESIGN.md R17): int_T g dS = A sum_a w_a g(q_a).
  RCS for a unit incident field: sigma_p = 4 pi r^2 |E_p|^2 = (k eta)^2 / (4 pi) |F . p^|^2,
  p^ in {theta^, phi^} of r^ (phi = 0 on the z axis).

A plain per-triangle-side loop over the basis functions, vectorised over bases; the phase
matrix per chunk of samples (a matmul serves as the sum over samples)."""
from __future__ import annotations

import numpy as np

# Dunavant degree-5 7-point rule on the reference triangle (barycentric, weights sum to 1)
_A, _B = 0.059715871789770, 0.470142064105115
_C, _D = 0.797426985353087, 0.101286507323456
BARY = np.array([[1 / 3, 1 / 3, 1 / 3], [_A, _B, _B], [_B, _A, _B], [_B, _B, _A],
                 [_C, _D, _D], [_D, _C, _D], [_D, _D, _C]])
WEIGHTS = np.array([0.225] + [0.132394152788506] * 3 + [0.125939180544827] * 3)


def rwg_samples(nodes, tris, tp, tm, vp, vm):
    """Sample positions q (N*14 x 3), real vectors g = A w_a f_n(q) (N*14 x 3) and basis
    index per sample: int f_n h dS = sum_samples g h(q)."""
    nodes = np.asarray(nodes, float)
    tris = np.asarray(tris)
    N = len(tp)
    # shared edge of T+ = its two vertices other than v+
    Tp = tris[tp]
    mask = Tp != np.asarray(vp)[:, None]
    edge = Tp[mask].reshape(N, 2)
    length = np.linalg.norm(nodes[edge[:, 0]] - nodes[edge[:, 1]], axis=1)
    pos, vec = [], []
    for T, v, sign in ((tp, vp, 1.0), (tm, vm, -1.0)):
        P = nodes[tris[T]]                                  # N x 3 vertices x 3
        area = 0.5 * np.linalg.norm(np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]), axis=1)
        for a in range(7):
            q = BARY[a, 0] * P[:, 0] + BARY[a, 1] * P[:, 1] + BARY[a, 2] * P[:, 2]
            f = sign * (length / (2 * area))[:, None] * (q - nodes[v])
            pos.append(q)
            vec.append(WEIGHTS[a] * area[:, None] * f)
    pos = np.stack(pos, 1).reshape(-1, 3)                   # basis-major: n * 14 + (side * 7 + a)
    vec = np.stack(vec, 1).reshape(-1, 3)
    idx = np.repeat(np.arange(N), 14)
    return pos, vec, idx


def farfield(nodes, tris, tp, tm, vp, vm, k, I, rhat, mono=False, chunk=50_000):
    """F (ndir x nrhs x 3) bistatic, or (ndir x 3) monostatic (direction d with column d)."""
    I = np.asarray(I, np.complex128)
    if I.ndim == 1:
        I = I[:, None]
    rhat = np.asarray(rhat, float)
    pos, vec, idx = rwg_samples(nodes, tris, tp, tm, vp, vm)
    ndir, nrhs = len(rhat), I.shape[1]
    F = np.zeros((ndir, 1 if mono else nrhs, 3), np.complex128)
    for s0 in range(0, len(pos), chunk):
        P = np.exp(1j * k * (rhat @ pos[s0:s0 + chunk].T))  # ndir x samples
        Is = I[idx[s0:s0 + chunk]]                          # samples x nrhs
        g = vec[s0:s0 + chunk]
        for x in range(3):
            if mono:
                F[:, 0, x] += np.einsum("ds,sd->d", P, g[:, x:x + 1] * Is)
            else:
                F[:, :, x] += P @ (g[:, x:x + 1] * Is)
    return F[:, 0, :] if mono else F


def sph_units(rhat):
    """theta^ and phi^ of each direction (phi = 0 on the z axis)."""
    rhat = np.asarray(rhat, float)
    st = np.hypot(rhat[:, 0], rhat[:, 1])
    ok = st > 1e-12
    cp = np.where(ok, rhat[:, 0] / np.where(ok, st, 1), 1.0)
    sp = np.where(ok, rhat[:, 1] / np.where(ok, st, 1), 0.0)
    th = np.stack([rhat[:, 2] * cp, rhat[:, 2] * sp, -st], 1)
    ph = np.stack([-sp, cp, 0 * cp], 1)
    return th, ph


def rcs(F, rhat, k, eta):
    """sigma (..., 2): (theta, phi) polarisation, m^2, from F (ndir x [nrhs x] 3)."""
    th, ph = sph_units(rhat)
    shp = (len(rhat),) + (1,) * (F.ndim - 2) + (3,)
    ft = (F * th.reshape(shp)).sum(-1)
    fp = (F * ph.reshape(shp)).sum(-1)
    c = (k * eta) ** 2 / (4 * np.pi)
    return np.stack([c * np.abs(ft) ** 2, c * np.abs(fp) ** 2], -1)
