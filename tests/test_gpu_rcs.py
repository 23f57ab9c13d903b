"""GPU parity of the far field / RCS post-processing (ps_farfield; SURVEY §8(f) NEXT-4,
PAPER.md:333-341) against the oracle (oracle/rcs.py): F per column relative L2 over the
directions <= 1e-11, sigma elementwise to 1e-10 of the column's peak; bistatic and
monostatic; ragged sizes (N, directions, columns not multiples of the tiles); the k = 0
closed form; the BASELINE monostatic sweeps of C2 (181) and C4 (360, sampled) on the
currents ps_solve returns."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from hmgen.build import CONFIGS, make_mesh, read_rhs, rwg_basis, plane_wave_dirs  # noqa: E402
from hmgen.synth import random_rhs                          # noqa: E402
from oracle.rcs import farfield as ff_ref, rcs as rcs_ref  # noqa: E402
from paper_2109_04129_b200 import PsError, farfield        # noqa: E402
from paper_2109_04129_b200.binding import PS_EINVAL        # noqa: E402

pytestmark = pytest.mark.gpu
ETA = 120 * np.pi
_mesh = {}


def _geom(name):
    if name not in _mesh:
        cfg = CONFIGS[name]
        m = make_mesh(cfg)
        _mesh[name] = (cfg, m, rwg_basis(m))
    return _mesh[name]


def _dirs(n, seed):
    v = np.random.default_rng(seed).standard_normal((n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _check(name, I, rh, mono, k=None):
    cfg, m, bs = _geom(name)
    k = cfg.k if k is None else k
    F, sig = farfield(m.nodes, m.tris, bs.tp, bs.tm, bs.vp, bs.vm, k, ETA, I, rh, mono=mono)
    F, sig = F.cpu().numpy(), sig.cpu().numpy()
    Fr = ff_ref(m.nodes, m.tris, bs.tp, bs.tm, bs.vp, bs.vm, k, I, rh, mono=mono)
    sr = rcs_ref(Fr, rh, k, ETA)
    if mono:
        F, Fr, sig, sr = F[:, None], Fr[:, None], sig[:, None], sr[:, None]
    for c in range(F.shape[1]):
        err = np.linalg.norm(F[:, c] - Fr[:, c]) / np.linalg.norm(Fr[:, c])
        assert err <= 1e-11, (c, err)
        assert np.abs(sig[:, c] - sr[:, c]).max() <= 1e-10 * sr[:, c].max()
    F2, _ = farfield(m.nodes, m.tris, bs.tp, bs.tm, bs.vp, bs.vm, k, ETA, I, rh, mono=mono)
    assert np.array_equal(F2.cpu().numpy().reshape(F.shape), F)        # deterministic
    return F, sig


def test_bistatic_c1():
    cfg, m, bs = _geom("C1")
    th = np.deg2rad(np.arange(0.0, 181.0, 1.0))
    rh = np.concatenate([np.stack([np.sin(th), 0 * th, np.cos(th)], 1), _dirs(40, 1),
                         [[0, 0, 1.0], [0, 0, -1.0]]])
    _check("C1", random_rhs(bs.N, 3, seed=2), rh, mono=False)       # 3 columns: ragged column tile
    _check("C1", random_rhs(bs.N, 9, seed=3), rh[:130], mono=False)


def test_monostatic_c1_and_ragged():
    cfg, m, bs = _geom("C1")
    for n in (1, 33, 129):
        _check("C1", random_rhs(bs.N, n, seed=n), _dirs(n, n + 1), mono=True)


def test_k0_closed_form_gpu():
    cfg, m, bs = _geom("C1")
    I = random_rhs(bs.N, 1, seed=4)[:, 0]
    P = m.nodes
    cp = P[m.tris[bs.tp]].mean(1)
    cm = P[m.tris[bs.tm]].mean(1)
    ref = ((bs.length / 2 * I)[:, None] * ((cp - P[bs.vp]) - (cm - P[bs.vm]))).sum(0)
    F, _ = farfield(m.nodes, m.tris, bs.tp, bs.tm, bs.vp, bs.vm, 0.0, ETA, I, _dirs(4, 5))
    F = F.cpu().numpy()[:, 0]
    assert np.abs(F - ref).max() <= 1e-12 * np.linalg.norm(ref)


def test_bad_arguments():
    cfg, m, bs = _geom("T0")
    I = random_rhs(bs.N, 2, seed=0)
    with pytest.raises(PsError) as e:
        farfield(m.nodes, m.tris, bs.tp, bs.tm, bs.vp, bs.vm, cfg.k, ETA, I, _dirs(3, 0), mono=True)
    assert e.value.status == PS_EINVAL
    F, s = farfield(m.nodes, m.tris, bs.tp, bs.tm, bs.vp, bs.vm, cfg.k, ETA, I, np.zeros((0, 3)))
    assert F.shape == (0, 2, 3)


def _solved_currents(cfgdata, name, cols):
    from paper_2109_04129_b200 import PsHandle
    import warnings
    meta = cfgdata(name)
    B, ang = read_rhs(meta["rhs"])
    h = PsHandle(meta["hm"])
    h.setup()
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().T
    Xd = torch.empty_like(Bd)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h.solve(Bd, Xd)
    h.close()
    return Xd, B


def test_monostatic_c2_sweep(cfgdata):
    """BASELINE config 1's 181-angle monostatic sweep on the solve's currents (RCS of the
    backscatter direction -k^ of each incidence)."""
    cfg, m, bs = _geom("C2")
    Xd, _ = _solved_currents(cfgdata, "C2", None)
    _, khat, _ = plane_wave_dirs(cfg)
    rh = -np.asarray(khat)
    I = Xd.cpu().numpy()
    _check("C2", np.asfortranarray(I), rh, mono=True)


@pytest.mark.slow
def test_monostatic_c4_sweep_sampled(cfgdata):
    """BASELINE config 3 (N = 96000): all 360 backscatter directions in one launch on the
    solve's currents; sampled columns against the oracle (columns are independent)."""
    cfg, m, bs = _geom("C4")
    Xd, _ = _solved_currents(cfgdata, "C4", None)
    _, khat, _ = plane_wave_dirs(cfg)
    rh = -np.asarray(khat)
    F, sig = farfield(m.nodes, m.tris, bs.tp, bs.tm, bs.vp, bs.vm, cfg.k, ETA, Xd, rh, mono=True)
    F = F.cpu().numpy()
    I = Xd.cpu().numpy()
    cols = [0, 1, 127, 179, 180, 255, 359]
    Fr = ff_ref(m.nodes, m.tris, bs.tp, bs.tm, bs.vp, bs.vm, cfg.k, I[:, cols], rh[cols], mono=True)
    err = np.linalg.norm(F[cols] - Fr, axis=1) / np.linalg.norm(Fr, axis=1)
    assert err.max() <= 1e-11, err
