"""Pins of the RCS oracle (oracle/rcs.py), no GPU:
an independent implementation (the generator's compiled far field), the k -> 0 closed form
of the RWG integrals, the translation phase law, monostatic = the diagonal of bistatic,
the spherical unit vectors, and the physics (C1 dense-LU currents vs the Mie series)."""
import numpy as np
import pytest

from hmgen.build import CONFIGS, EfieLib, make_mesh, rwg_basis
from hmgen.synth import random_rhs
from oracle.rcs import farfield, rcs, sph_units
from tests.mie import mie_eplane_rcs

ETA = 120 * np.pi


@pytest.fixture(scope="module")
def c1():
    cfg = CONFIGS["C1"]
    mesh = make_mesh(cfg)
    bs = rwg_basis(mesh)
    return cfg, mesh, bs


def _dirs(n, seed):
    v = np.random.default_rng(seed).standard_normal((n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _ff(mesh, bs, k, I, rh, mono=False):
    return farfield(mesh.nodes, mesh.tris, bs.tp, bs.tm, bs.vp, bs.vm, k, I, rh, mono=mono)


def test_matches_generator_farfield(c1):
    """Same definition, independent code (hmgen/csrc/efie.cpp efie_farfield, C++)."""
    cfg, mesh, bs = c1
    I = random_rhs(bs.N, 2, seed=1)
    rh = _dirs(23, 0)
    F = _ff(mesh, bs, cfg.k, I, rh)
    ef = EfieLib(mesh, bs, cfg.k)
    for c in range(2):
        G = ef.farfield(I[:, c], rh)
        assert np.linalg.norm(F[:, c] - G) <= 1e-12 * np.linalg.norm(G)


def test_k0_closed_form(c1):
    """k = 0: the 7-point rule is exact on the linear f_n, int_{T+-} f_n = +-l_n/2 (c+- - v+-)
    with c the centroid, so F = sum_n I_n l_n / 2 ((c+ - v+) - (c- - v-)) for every r^."""
    _, mesh, bs = c1
    I = random_rhs(bs.N, 1, seed=2)[:, 0]
    P = mesh.nodes
    cp = P[mesh.tris[bs.tp]].mean(1)
    cm = P[mesh.tris[bs.tm]].mean(1)
    ref = ((bs.length / 2 * I)[:, None] * ((cp - P[bs.vp]) - (cm - P[bs.vm]))).sum(0)
    F = _ff(mesh, bs, 0.0, I, _dirs(5, 3))
    for d in range(5):
        assert np.linalg.norm(F[d, 0] - ref) <= 1e-12 * np.linalg.norm(ref)


def test_translation_phase(c1):
    """Moving the body by t multiplies F(r^) by exp(+j k r^.t) (the far-zone phase)."""
    cfg, mesh, bs = c1
    I = random_rhs(bs.N, 1, seed=4)
    rh = _dirs(7, 5)
    t = np.array([0.3, -1.1, 0.45])
    F0 = _ff(mesh, bs, cfg.k, I, rh)
    moved = type(mesh)(mesh.nodes + t, mesh.tris)
    F1 = _ff(moved, bs, cfg.k, I, rh)
    ref = F0 * np.exp(1j * cfg.k * (rh @ t))[:, None, None]
    assert np.linalg.norm(F1 - ref) <= 1e-12 * np.linalg.norm(ref)


def test_monostatic_is_bistatic_diagonal(c1):
    cfg, mesh, bs = c1
    I = random_rhs(bs.N, 6, seed=6)
    rh = _dirs(6, 7)
    Fb = _ff(mesh, bs, cfg.k, I, rh)
    Fm = _ff(mesh, bs, cfg.k, I, rh, mono=True)
    assert np.allclose(Fm, Fb[np.arange(6), np.arange(6)], rtol=1e-13, atol=0)
    sb = rcs(Fb, rh, cfg.k, ETA)
    sm = rcs(Fm, rh, cfg.k, ETA)
    assert np.allclose(sm, sb[np.arange(6), np.arange(6)], rtol=1e-12)


def test_spherical_units():
    rh = np.concatenate([_dirs(50, 8), [[0, 0, 1.0], [0, 0, -1.0], [1.0, 0, 0]]])
    th, ph = sph_units(rh)
    for a, b in ((th, ph), (th, rh), (ph, rh)):
        assert np.abs((a * b).sum(1)).max() < 1e-14
    assert np.allclose(np.linalg.norm(th, axis=1), 1) and np.allclose(np.linalg.norm(ph, axis=1), 1)
    assert np.allclose(np.cross(rh, th), ph)                       # right-handed (r^, theta^, phi^)


def test_mie_bistatic_rcs_c1(cfgdata, c1):
    """Physics: dense-LU currents of the file's Z on C1, E-plane bistatic RCS from this oracle
    vs the PEC-sphere Mie series within 1.5 dB (samples > 30 dB below the peak excluded)."""
    from hmgen.build import read_rhs
    from oracle import read_hm
    from oracle.dense import dense_ZF, dense_ZN, direct_solve
    cfg, mesh, bs = c1
    meta = cfgdata("C1")
    H = read_hm(meta["hm"])
    B, _ = read_rhs(meta["rhs"])
    x = direct_solve(dense_ZN(H) + dense_ZF(H), B[:, 0])
    th = np.deg2rad(np.arange(0.0, 181.0, 2.0))
    rh = np.stack([np.sin(th), 0 * th, np.cos(th)], 1)
    sig = rcs(_ff(mesh, bs, cfg.k, x, rh), rh, cfg.k, ETA)[:, 0, 0]
    ref = mie_eplane_rcs(cfg.k * 0.5, cfg.lam, np.pi - th)
    d_db = 10 * np.log10(sig) - 10 * np.log10(ref)
    keep = 10 * np.log10(ref) > 10 * np.log10(ref.max()) - 30
    assert np.abs(d_db[keep]).max() <= 1.5
