"""Pins of the INPUT GENERATOR (hmgen): mesh/RWG counts, analytic singular
integrals, EFIE symmetry, ACA accuracy (Eq. 12) and Mie agreement
(§V.C.1). CPU only."""
import math

import numpy as np
import pytest

from hmgen.build import (CONFIGS, EfieLib, build_tree, cube_mesh, cylinder_mesh, icosphere,
                         make_mesh, nd_order, potential_integrals, rwg_basis, plane_wave_dirs,
                         checksum64)
from tests.mie import mie_eplane_rcs


def test_icosphere_counts():
    # icosahedron 12/20/30; one subdivision 42/80/120
    m0 = icosphere(1.0, 0)
    assert (len(m0.nodes), len(m0.tris), rwg_basis(m0).N) == (12, 20, 30)
    m1 = icosphere(1.0, 1)
    assert (len(m1.nodes), len(m1.tris), rwg_basis(m1).N) == (42, 80, 120)
    m3 = icosphere(0.5, 3)
    assert (len(m3.tris), rwg_basis(m3).N) == (1280, 1920)      # BASELINE config 0
    assert np.allclose(np.linalg.norm(m3.nodes, axis=1), 0.5, atol=1e-12)


def test_cube_and_cylinder_closed():
    c = cube_mesh(1.0, 1)
    assert (len(c.tris), rwg_basis(c).N) == (12, 18)
    c30 = cube_mesh(3.0, 30)
    assert (len(c30.tris), rwg_basis(c30).N) == (10800, 16200)    # BASELINE config 1
    cy = cylinder_mesh(1.0, 2.0, 0.25)
    b = rwg_basis(cy)
    assert b.N == 3 * len(cy.tris) // 2                            # closed: every edge interior


def _brute_potential(tri, r, n=300):
    # midpoint rule on a fine barycentric grid
    acc_s, acc_v = 0.0, np.zeros(3)
    p0, p1, p2 = tri
    area = 0.5 * np.linalg.norm(np.cross(p1 - p0, p2 - p0))
    cnt = 0
    for i in range(n):
        for j in range(n - i):
            for up in (0, 1):
                if up == 1 and i + j + 1 >= n:
                    continue
                if up == 0:
                    a, b = (i + 1 / 3) / n, (j + 1 / 3) / n
                else:
                    a, b = (i + 2 / 3) / n, (j + 2 / 3) / n
                q = p0 + a * (p1 - p0) + b * (p2 - p0)
                d = q - r
                R = np.linalg.norm(d)
                acc_s += 1 / R
                acc_v += d / R
                cnt += 1
    return acc_s * area / cnt, acc_v * area / cnt


@pytest.mark.parametrize("r", [[0.3, 0.2, 0.5], [1.4, -0.3, 0.0], [0.2, 0.9, -0.2]])
def test_potential_integrals_vs_quadrature(r):
    tri = np.array([[0.0, 0.0, 0.0], [1.0, 0.1, 0.0], [0.2, 0.8, 0.1]])
    js, jv = potential_integrals(tri, np.array(r))
    bs, bv = _brute_potential(tri, np.array(r), n=160)
    assert abs(js - bs) / abs(bs) < 2e-4
    assert np.linalg.norm(jv - bv) / np.linalg.norm(bv) < 2e-4


def test_potential_singular_point_inside():
    # observation point inside the triangle (R -> 0 integrable singularity):
    # Int 1/R over an equilateral triangle seen from its centroid has the closed form
    # 3 h ln((1 + sin 60)/(cos 60 ... )) ; use the polar form 3 * Int_{-pi/3}^{pi/3} h/cos t dt
    s = 1.0
    tri = np.array([[0, 0, 0], [s, 0, 0], [s / 2, s * math.sqrt(3) / 2, 0]])
    c = tri.mean(0)
    h = s / (2 * math.sqrt(3))        # inradius
    exact = 3 * h * 2 * math.log(math.tan(math.pi / 4 + math.pi / 6))
    js, _ = potential_integrals(tri, c)
    assert abs(js - exact) < 1e-12


def test_efie_symmetry_and_block_structure():
    cfg = CONFIGS["T1"]
    mesh = make_mesh(cfg)
    basis = rwg_basis(mesh)
    ef = EfieLib(mesh, basis, cfg.k)
    idx = np.arange(basis.N)
    Z = ef.block(idx, idx)
    # Galerkin EFIE is complex-symmetric; one-sided singular
    # extraction breaks exact symmetry only on touching pairs
    touching = np.zeros_like(Z, dtype=bool)
    tri_of = [set(mesh.tris[basis.tp[m]]) | set(mesh.tris[basis.tm[m]]) for m in range(basis.N)]
    for m in range(basis.N):
        for n in range(basis.N):
            touching[m, n] = bool(tri_of[m] & tri_of[n])
    rel = np.abs(Z - Z.T) / np.abs(Z).max()
    assert rel[~touching].max() < 1e-12
    assert rel.max() < 2e-3


def test_tree_tiling_and_near_degree():
    """Every leaf pair is covered exactly once by a near block or a far block."""
    rng = np.random.default_rng(3)
    pts = rng.uniform(0, 2, size=(600, 3))
    t = build_tree(pts, 0.25)
    N = 600
    cover = np.zeros((N, N), dtype=np.int32)
    lo = t.leaf_off
    for i, j in t.near:
        cover[lo[i]:lo[i + 1], lo[j]:lo[j + 1]] += 1
        if i != j:
            cover[lo[j]:lo[j + 1], lo[i]:lo[i + 1]] += 1
    for r0, m, c0, n, _ in t.far:
        cover[r0:r0 + m, c0:c0 + n] += 1
        cover[c0:c0 + n, r0:r0 + m] += 1
    assert (cover == 1).all()
    deg = np.bincount(t.near.ravel(), minlength=len(lo) - 1)
    assert deg.max() <= 28          # 26 neighbours + self counted twice in (i,i)


def test_nd_order_is_permutation_and_separates():
    rng = np.random.default_rng(5)
    ijk = np.unique(rng.integers(0, 8, size=(300, 3)), axis=0)
    o = nd_order(ijk)
    assert sorted(o.tolist()) == list(range(len(ijk)))


def test_checksum_sensitivity():
    a = np.arange(1000, dtype=np.int64)
    h = checksum64(a.tobytes())
    b = a.copy()
    b[[3, 4]] = b[[4, 3]]
    assert checksum64(b.tobytes()) != h


def test_aca_matches_dense_entries(cfgdata):
    """PAPER.md Eq. (12): ||Z_sub - A B||_F <= eps ||Z_sub||_F per far block.
    The ACA stopping rule is an estimate (R18), so the pin allows 3 eps
    per block and requires the median below eps."""
    from oracle import read_hm
    cfg = CONFIGS["C1"]
    meta = cfgdata("C1")
    H = read_hm(meta["hm"])
    mesh = make_mesh(cfg)
    basis = rwg_basis(mesh)
    ef = EfieLib(mesh, basis, cfg.k)
    errs = []
    for (r0, m, c0, n, lev, U, V) in H.far[::3]:
        Z = ef.block(H.perm[r0:r0 + m], H.perm[c0:c0 + n])
        errs.append(np.linalg.norm(Z - U @ V.T) / np.linalg.norm(Z))
    errs = np.array(errs)
    assert errs.max() <= 3 * cfg.aca_eps
    assert np.median(errs) <= cfg.aca_eps


def test_near_blocks_match_entries(cfgdata):
    from oracle import read_hm
    cfg = CONFIGS["C1"]
    H = read_hm(cfgdata("C1")["hm"])
    mesh = make_mesh(cfg)
    basis = rwg_basis(mesh)
    ef = EfieLib(mesh, basis, cfg.k)
    lo, P = H.leaf_off, H.perm
    for i, j, Z in H.near[::17]:
        ref = ef.block(P[lo[i]:lo[i + 1]], P[lo[j]:lo[j + 1]])
        if i == j:
            assert np.array_equal(Z, Z.T)                       # exact symmetry by construction
            iu = np.triu_indices(Z.shape[0])
            assert np.allclose(Z[iu], ref[iu], rtol=0, atol=1e-13 * np.abs(ref).max())
        else:
            assert np.allclose(Z, ref, rtol=0, atol=1e-13 * np.abs(ref).max())


def test_mie_bistatic_rcs_c1(cfgdata):
    """Physics pin (BASELINE config 0): dense-LU solution of the file's Z = Z_N + Z_F,
    bistatic E-plane RCS vs the PEC-sphere Mie series: mean |dsigma| <= 1.5 dB
    excluding samples > 30 dB below the peak."""
    from oracle import read_hm
    from oracle.dense import dense_ZF, dense_ZN, direct_solve
    from hmgen.build import read_rhs
    cfg = CONFIGS["C1"]
    meta = cfgdata("C1")
    H = read_hm(meta["hm"])
    B, _ = read_rhs(meta["rhs"])
    x = direct_solve(dense_ZN(H) + dense_ZF(H), B[:, 0])
    mesh = make_mesh(cfg)
    ef = EfieLib(mesh, rwg_basis(mesh), cfg.k)
    th = np.deg2rad(np.arange(0.0, 181.0, 2.0))
    rh = np.stack([np.sin(th), 0 * th, np.cos(th)], 1)
    thh = np.stack([np.cos(th), 0 * th, -np.sin(th)], 1)
    F = ef.farfield(x, rh)
    eta = 120 * np.pi
    sig = (cfg.k * eta) ** 2 / (4 * np.pi) * np.abs((F * thh).sum(1)) ** 2
    # incidence along -z: scattering angle = pi - theta
    ref = mie_eplane_rcs(cfg.k * 0.5, cfg.lam, np.pi - th)
    d_db = 10 * np.log10(sig) - 10 * np.log10(ref)
    keep = 10 * np.log10(ref) > 10 * np.log10(ref.max()) - 30
    assert np.abs(d_db[keep]).mean() <= 1.5
    assert np.abs(d_db[keep]).max() <= 1.5


def test_plane_wave_table():
    ang, kh, ep = plane_wave_dirs(CONFIGS["C4"])
    assert ang.shape == (360, 2)
    assert np.allclose(np.abs(np.einsum("ij,ij->i", kh, ep.real)), 0, atol=1e-12)   # transverse
    assert np.allclose(np.linalg.norm(ep, axis=1), 1)


def test_c4_cylinder_mesh_matches_baseline():
    """BASELINE configs[3]: closed cylinder r=1 m, L=10 m at 600 MHz, MEAN edge lambda/10
    over all edges, ~64k triangles, N ~ 96k."""
    from hmgen.build import make_mesh, mean_edge
    cfg = CONFIGS["C4"]
    m = make_mesh(cfg)
    assert abs(mean_edge(m) / (cfg.lam / 10) - 1) < 0.01
    assert 62000 <= len(m.tris) <= 66000
    b = rwg_basis(m)
    assert b.N == 3 * len(m.tris) // 2 and 93000 <= b.N <= 99000
