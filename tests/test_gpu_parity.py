"""GPU parity: libps (sm_100a kernels, through the C ABI) vs the oracle.

Bar (BASELINE.json north_star): per RHS column, relative L2 <= 1e-11 (complex128).
Each hot-path step is checked on its own through ps_apply (R^T, D^-1, R, Z_F,
U), then the whole ps_solve, on physical configs (T1, C1, T2, and the bench
config C2 at its full 181 RHS) and on seeded synthetic systems that cover the
edge cases: size-1 leaves and ragged leaf sizes, a single leaf, no far field,
nrhs = 1 and ragged column tiles, host and device buffers.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from hmgen.build import read_rhs                             # noqa: E402
from hmgen.synth import random_rhs                          # noqa: E402
from oracle import (apply_Dinv, apply_R, apply_Rt, apply_U, apply_ZF, compute_scaling,  # noqa: E402
                    read_hm, solve)
from paper_2109_04129_b200 import (PS_OP_DINV, PS_OP_R, PS_OP_RT, PS_OP_U, PS_OP_ZF,  # noqa: E402
                                   PsError, PsHandle)
from paper_2109_04129_b200.binding import PS_EDIVERGED, PS_ESTATE, PS_EINVAL, PS_ESINGULAR  # noqa: E402
from tests.conftest import rel_l2_cols                      # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-11


def _dev(A):
    """column-major complex128 CUDA tensor from a numpy N x nrhs array"""
    A = np.asfortranarray(A, dtype=np.complex128)
    return torch.from_numpy(np.ascontiguousarray(A.T)).cuda().T


def _host(T):
    return np.asfortranarray(T.T.cpu().numpy().T)


_cache = {}


def _load(path):
    if path not in _cache:
        H = read_hm(path)
        S = compute_scaling(H)
        h = PsHandle(path)
        h.setup()
        _cache[path] = (H, S, h)
    return _cache[path]


def _ops_check(path, nrhs, seed=0):
    H, S, h = _load(path)
    X = random_rhs(H.N, nrhs, seed)
    Xd = _dev(X)
    Y = torch.empty_like(Xd)
    e = S.e2rwg
    xe = X[e]
    ref = {
        PS_OP_RT: apply_Rt(S, xe),
        PS_OP_DINV: apply_Dinv(S, xe),
        PS_OP_R: apply_R(S, xe),
        PS_OP_ZF: apply_ZF(H, S, xe),
        PS_OP_U: apply_U(H, S, xe),
    }
    for op, r in ref.items():
        h.apply(op, Xd, Y)
        y = _host(Y)[e]
        err = rel_l2_cols(y, r)
        assert err.max() <= TOL, (op, err.max())


def _solve_check(path, B, check_host=True):
    H, S, h = _load(path)
    ref = solve(H, S, B)
    Bd = _dev(B)
    Xd = torch.empty_like(Bd)
    st, rep = h.solve(Bd, Xd)
    x = _host(Xd)
    err = rel_l2_cols(x, ref.x)
    assert err.max() <= TOL, err.max()
    assert np.allclose(rep["it0"], ref.it0, rtol=1e-11)
    assert np.allclose(rep["it1"], ref.it1, rtol=1e-10)
    assert (st == PS_EDIVERGED) == (ref.status == "diverged")
    assert rep["n_diverged"] == int((ref.ratio >= 0.1).sum())
    if check_host:
        Xh = np.zeros_like(np.asfortranarray(B))
        h.solve(np.asfortranarray(B), Xh)
        assert np.array_equal(Xh, x)              # same kernels, bitwise
    # determinism: a second solve is bitwise identical
    X2 = torch.empty_like(Bd)
    h.solve(Bd, X2)
    assert torch.equal(X2, Xd)
    return err, rep


@pytest.mark.parametrize("name", ["T1", "C1", "T2"])
def test_ops_physical(cfgdata, name):
    _ops_check(cfgdata(name)["hm"], nrhs=3)


@pytest.mark.parametrize("kw", [dict(n_points=500, seed=3, clustered=True),
                                dict(n_points=700, seed=4),
                                dict(n_points=2500, seed=5, leaf_edge=0.15)])
def test_ops_synthetic(synthfile, kw):
    _ops_check(synthfile(**kw)[0], nrhs=5)


def test_dinv_blocks(cfgdata):
    H, S, h = _load(cfgdata("C1")["hm"])
    for pos in range(S.n):
        D = h.dinv(pos)
        ref = S.Dinv[pos]
        assert np.linalg.norm(D - ref) <= 1e-12 * np.linalg.norm(ref)
        assert h.elim_leaf(pos) == S.leaf_of[pos]


@pytest.mark.parametrize("nrhs", [1, 33])
def test_solve_c1(cfgdata, nrhs):
    meta = cfgdata("C1")
    H, S, h = _load(meta["hm"])
    B0, _ = read_rhs(meta["rhs"])
    B = np.asfortranarray(np.concatenate([B0, random_rhs(H.N, nrhs - 1, 7)], 1) if nrhs > 1 else B0)
    _solve_check(meta["hm"], B)


@pytest.mark.parametrize("nrhs", [1, 40])
def test_solve_async_matches_solve(cfgdata, nrhs):
    """ps_solve_async queues the same kernels without a host sync: three solves pipelined on
    one stream (different inputs, one workspace) equal the synchronous solves bitwise, and
    ps_solve_report returns the last one's norms / status; the result also meets the oracle bar."""
    meta = cfgdata("C1")
    H, S, h = _load(meta["hm"])
    st = torch.cuda.Stream()
    Bs = [_dev(random_rhs(H.N, nrhs, 20 + i)) for i in range(3)]
    Xs = [torch.empty_like(b) for b in Bs]
    Xa = [torch.empty_like(b) for b in Bs]
    reps = [h.solve(b, x)[1] for b, x in zip(Bs, Xs)]
    st.wait_stream(torch.cuda.current_stream())
    with pytest.raises(PsError) as ei:          # nothing pending yet
        h.solve_report()
    assert ei.value.status == PS_ESTATE
    for b, x in zip(Bs, Xa):
        h.solve_async(b, x, stream=st)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        status, rep = h.solve_report()
    for x, y in zip(Xs, Xa):
        assert torch.equal(x, y)
    assert np.array_equal(rep["it0"], reps[-1]["it0"]) and np.array_equal(rep["it1"], reps[-1]["it1"])
    assert rep["n_diverged"] == reps[-1]["n_diverged"] and (status == PS_EDIVERGED) == (rep["n_diverged"] > 0)
    ref = solve(H, S, _host(Bs[-1]))
    assert rel_l2_cols(_host(Xa[-1]), ref.x).max() <= TOL
    assert np.allclose(rep["ratio"], ref.ratio, rtol=1e-10)


def test_solve_t2_plane_waves(cfgdata):
    meta = cfgdata("T2")
    B, _ = read_rhs(meta["rhs"])
    _solve_check(meta["hm"], B)


def test_solve_synthetic_convergent(synthfile):
    p, _ = synthfile(n_points=900, seed=8, far_scale=0.05)
    H, S, h = _load(p)
    err, rep = _solve_check(p, random_rhs(H.N, 40, 9))
    assert rep["n_diverged"] == 0


def test_solve_single_leaf_and_no_far(synthfile):
    p, hd = synthfile(n_points=30, box=0.2, leaf_edge=0.25, seed=2)
    assert hd.stats["n_leaves"] == 1 and hd.stats["n_far"] == 0
    H, S, h = _load(p)
    _solve_check(p, random_rhs(H.N, 2, 1))
    p2, hd2 = synthfile(n_points=120, box=0.5, leaf_edge=0.25, seed=3)
    assert hd2.stats["n_far"] == 0
    _solve_check(p2, random_rhs(hd2.N, 3, 2))


@pytest.mark.slow
def test_solve_c2_bench_config_full(cfgdata):
    """The bench workload (BASELINE config 1, 181 RHS) compared on every column."""
    meta = cfgdata("C2")
    B, _ = read_rhs(meta["rhs"])
    _solve_check(meta["hm"], B, check_host=False)


def test_error_paths(synthfile, tmp_path):
    p, hd = synthfile(n_points=200, seed=11)
    h = PsHandle(p)
    B = _dev(random_rhs(hd.N, 1, 0))
    X = torch.empty_like(B)
    with pytest.raises(PsError) as e:
        h.solve(B, X)
    assert e.value.status == PS_ESTATE
    h.setup()
    with pytest.raises(PsError) as e:
        h.setup()
    assert e.value.status == PS_ESTATE
    with pytest.raises(PsError) as e:
        h.solve(B, B)                     # X aliases B
    assert e.value.status == PS_EINVAL
    h.close()


def test_singular_leaf_is_named(tmp_path):
    from hmgen.build import write_hm
    from hmgen.synth import synthetic
    hd = synthetic(n_points=200, seed=12)
    # zero the diagonal block of leaf 0 -> exactly singular at its elimination
    i, j, off = hd.near_list[0]
    assert i == j == 0
    n0 = int(hd.tree.leaf_off[1] - hd.tree.leaf_off[0])
    hd.near_arena[off:off + n0 * n0] = 0
    # decouple leaf 0 so no Schur update can make it regular again
    for b, (a, c, o) in enumerate(hd.near_list):
        if a == 0 and c != 0:
            nc = int(hd.tree.leaf_off[c + 1] - hd.tree.leaf_off[c])
            hd.near_arena[o:o + n0 * nc] = 0
    p = str(tmp_path / "sing.hm")
    write_hm(p, hd)
    h = PsHandle(p)
    with pytest.raises(PsError) as e:
        h.setup()
    assert e.value.status == PS_ESINGULAR
    assert "(leaf 0)" in str(e.value)


@pytest.mark.slow
def test_ops_c3(cfgdata):
    """BASELINE config 2 (sphere N=30720, 113-unknown leaves: row tiles 32+32+32+17)."""
    _ops_check(cfgdata("C3")["hm"], nrhs=2)


@pytest.mark.slow
def test_solve_c3_plane_waves(cfgdata):
    meta = cfgdata("C3")
    B, _ = read_rhs(meta["rhs"])
    _solve_check(meta["hm"], np.asfortranarray(B[:, :181]), check_host=False)
    _solve_check(meta["hm"], np.asfortranarray(B[:, :1]), check_host=True)     # the 1-RHS run


@pytest.mark.slow
def test_solve_c4_plane_waves(cfgdata):
    """BASELINE config 3 (closed cylinder, N=96000, 5184 leaves of mean 18.5 unknowns):
    both polarisations, a few monostatic angles, plus R^T/R/Z_F."""
    meta = cfgdata("C4")
    B, _ = read_rhs(meta["rhs"])
    cols = [0, 90, 180, 270]                 # theta-pol and phi-pol incidences
    _solve_check(meta["hm"], np.asfortranarray(B[:, cols]), check_host=False)
    _ops_check(meta["hm"], nrhs=2)


@pytest.mark.slow
def test_solve_c4_bench_config_sampled(cfgdata):
    """BASELINE config 3 in the bench's launch configuration (all 360 RHS in one solve:
    wide tiles, the single-launch program), checked on sampled columns the oracle
    solves one by one (columns are independent problems)."""
    meta = cfgdata("C4")
    B, _ = read_rhs(meta["rhs"])
    H, S, h = _load(meta["hm"])
    Bd = _dev(np.asfortranarray(B))
    Xd = torch.empty_like(Bd)
    st, rep = h.solve(Bd, Xd)
    x = _host(Xd)
    # at least one column in each of the six 64-column tiles (0-63, ..., 320-359), the
    # polarisation switch (179 / 180) and the ragged last tile's last column
    cols = [0, 1, 63, 64, 100, 128, 179, 180, 181, 192, 255, 256, 300, 320, 359]
    ref = solve(H, S, np.asfortranarray(B[:, cols]))
    err = rel_l2_cols(x[:, cols], ref.x)
    assert err.max() <= TOL, err.max()
    assert np.allclose(rep["it0"][cols], ref.it0, rtol=1e-11)
    assert np.allclose(rep["it1"][cols], ref.it1, rtol=1e-10)
    # the e2e path of the bench: host buffers, two pipelined 180-column halves
    Xh = np.zeros_like(np.asfortranarray(B))
    _, reph = h.solve(np.asfortranarray(B), Xh)
    assert rel_l2_cols(Xh[:, cols], ref.x).max() <= TOL
    assert np.allclose(reph["it0"], rep["it0"], rtol=1e-12) and np.allclose(reph["it1"], rep["it1"], rtol=1e-12)
    assert reph["n_diverged"] == rep["n_diverged"]


@pytest.mark.parametrize("nrhs", [8, 9, 63, 64, 65, 128, 129, 200])
def test_solve_column_tile_boundaries(cfgdata, nrhs):
    """nrhs at and around the narrow / wide column-tile edges (8, 64): ragged last
    tiles, the narrow -> wide switch, several column tiles per task."""
    meta = cfgdata("C1")
    H, S, h = _load(meta["hm"])
    B = random_rhs(H.N, nrhs, 17)
    Bd = _dev(B)
    Xd = torch.empty_like(Bd)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st, rep = h.solve(Bd, Xd)
    ref = solve(H, S, B)
    assert rel_l2_cols(_host(Xd), ref.x).max() <= TOL
    assert np.allclose(rep["it0"], ref.it0, rtol=1e-11)


@pytest.mark.parametrize("which", ["C1", "synth"])
def test_rcm_ordering(cfgdata, synthfile, which):
    """ps_setup ordering = 2 (reverse Cuthill-McKee, recomputed by libps): x is the
    order-invariant two-term solution (oracle in the file's ND order), it_0 / it_1
    are those of the oracle run in libps's RCM order (read back with ps_elim_leaf)."""
    path = cfgdata("C1")["hm"] if which == "C1" else synthfile(n_points=900, seed=7, clustered=True)[0]
    H = read_hm(path)
    h = PsHandle(path)
    h.setup(ordering=2)
    order = np.array([h.elim_leaf(p) for p in range(H.n_leaves)])
    assert sorted(order.tolist()) == list(range(H.n_leaves))
    assert not np.array_equal(order, H.elim)              # a different order really is used
    B = random_rhs(H.N, 3, 9)
    Bd = _dev(B)
    Xd = torch.empty_like(Bd)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st, rep = h.solve(Bd, Xd)
    ref_nd = solve(H, compute_scaling(H), B)
    ref_rcm = solve(H, compute_scaling(H, order), B)
    assert rel_l2_cols(_host(Xd), ref_nd.x).max() <= TOL
    assert rel_l2_cols(_host(Xd), ref_rcm.x).max() <= TOL
    assert np.allclose(rep["it0"], ref_rcm.it0, rtol=1e-11)
    assert np.allclose(rep["it1"], ref_rcm.it1, rtol=1e-10)
    h.close()
