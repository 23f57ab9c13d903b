"""BASELINE config 4 (PEC sphere r = 3 m, icosphere sub-7, N = 491520) on the GPU.

The oracle's sequential scaling cannot run at this size, so parity is pinned by
properties that hold at any size (SURVEY §8(c) "residual pins"), using the
file's own near field Z_N on the host (numpy block mat-vec, independent of libps):

  * y0 = R D^-1 R^T b (GPU, ps_apply) solves the near field:  Z_N y0 = b;
  * x  = the two-term solution (ps_solve) satisfies        Z_N x  = b - Z_F y0
    with t = Z_F y0 from ps_apply — i.e. x = Z_N^-1 b - Z_N^-1 Z_F Z_N^-1 b
    (Appendix B of SURVEY.md), to rounding.

Generation takes minutes of CPU and tens of GB of host memory, so the test runs
only when PS_C5=1 (the driver's default GPU run skips it).
"""
import os

import numpy as np
import pytest

_c5 = [pytest.mark.gpu, pytest.mark.slow,
       pytest.mark.skipif(os.environ.get("PS_C5") != "1", reason="set PS_C5=1 (minutes of CPU, tens of GB)")]


def _near_apply(H, x):
    """Z_N x for RWG-ordered x (N x nrhs), from the file's symmetric near blocks."""
    xm = x[H.perm]                        # Morton order
    ym = np.zeros_like(xm)
    off = H.leaf_off
    for i, j, Z in H.near:
        a0, a1, b0, b1 = off[i], off[i + 1], off[j], off[j + 1]
        ym[a0:a1] += Z @ xm[b0:b1]
        if i != j:
            ym[b0:b1] += Z.T @ xm[a0:a1]
    y = np.empty_like(ym)
    y[H.perm] = ym
    return y


def test_near_apply_is_the_near_field(cfgdata):
    """The host Z_N mat-vec used below equals the dense near field (C1, CPU)."""
    from oracle import read_hm
    from oracle.dense import dense_ZN
    H = read_hm(cfgdata("C1")["hm"])
    rng = np.random.default_rng(0)
    x = rng.standard_normal((H.N, 2)) + 1j * rng.standard_normal((H.N, 2))
    ZN = dense_ZN(H)
    assert np.linalg.norm(_near_apply(H, x) - ZN @ x) <= 1e-13 * np.linalg.norm(ZN @ x)


@pytest.mark.parametrize("m", [0], ids=["C5"])
@_c5[0]
@_c5[1]
@_c5[2]
def test_c5_residual_pins(m):
    import warnings
    torch = pytest.importorskip("torch")
    from hmgen.build import load_or_generate, read_rhs
    from oracle import read_hm
    from paper_2109_04129_b200 import PS_OP_DINV, PS_OP_R, PS_OP_RT, PS_OP_ZF, PsHandle
    from tests.conftest import rel_l2_cols
    meta = load_or_generate("C5")
    B, _ = read_rhs(meta["rhs"])
    B = np.asfortranarray(B[:, :2])
    h = PsHandle(meta["hm"])
    h.setup()

    def dev(A):
        return torch.from_numpy(np.ascontiguousarray(np.asfortranarray(A).T)).cuda().T

    def host(T):
        return np.asfortranarray(T.T.cpu().numpy().T)

    Bd = dev(B)
    Xd = torch.empty_like(Bd)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h.solve(Bd, Xd)
    t1, t2, y0 = torch.empty_like(Bd), torch.empty_like(Bd), torch.empty_like(Bd)
    h.apply(PS_OP_RT, Bd, t1)
    h.apply(PS_OP_DINV, t1, t2)
    h.apply(PS_OP_R, t2, y0)
    tF = torch.empty_like(Bd)
    h.apply(PS_OP_ZF, y0, tF)
    x, y0h, tFh = host(Xd), host(y0), host(tF)
    h.close()
    H = read_hm(meta["hm"])
    r0 = rel_l2_cols(_near_apply(H, y0h), B)
    r1 = np.linalg.norm(_near_apply(H, x) - (B - tFh), axis=0) / np.linalg.norm(B, axis=0)
    print(f"C5 N={H.N}: ||Z_N y0 - b||/||b|| = {r0.max():.3e}, ||Z_N x - (b - Z_F y0)||/||b|| = {r1.max():.3e}")
    assert r0.max() <= 1e-9, r0
    assert r1.max() <= 1e-9, r1
