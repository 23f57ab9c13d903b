"""GPU parity of the row-partitioned solve (SURVEY §8(e) option 1).

One GPU: the ranks of a row partition are handles of one process solved by
ps_solve_group — every rank's own tables and workspace, the same phases and
exchange ranges as the NCCL path, run in rank order with device copies as the
collectives. Bar: per RHS column relative L2 <= 1e-11 against the oracle
(BASELINE.json north_star), the norms of Eq. 44 to 1e-11.

With >= 2 GPUs, test_nccl_two_ranks launches two processes that solve through
NCCL (skipped on a single-GPU box).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from hmgen.synth import random_rhs                          # noqa: E402
from oracle import compute_scaling, read_hm, solve           # noqa: E402
from paper_2109_04129_b200 import PsError, PsHandle, solve_group  # noqa: E402
from paper_2109_04129_b200.binding import setup_group             # noqa: E402
from paper_2109_04129_b200.binding import PS_ESTATE, PS_EINVAL    # noqa: E402
from tests.conftest import rel_l2_cols                      # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-11


def _dev(A):
    A = np.asfortranarray(A, dtype=np.complex128)
    return torch.from_numpy(np.ascontiguousarray(A.T)).cuda().T


def _host(T):
    return np.asfortranarray(T.T.cpu().numpy().T)


def _group(path, P):
    """P in-process ranks with the sharded setup (ps_setup_group: each rank factors its
    own interior subtrees and the separators; separator rows summed over the ranks)."""
    hs = [PsHandle(path, device=0, rank=g, nranks=P, partition=True) for g in range(P)]
    setup_group(hs)
    return hs


def _check(path, P, nrhs, seed=3):
    H = read_hm(path)
    S = compute_scaling(H)
    B = random_rhs(H.N, nrhs, seed)
    ref = solve(H, S, B)
    hs = _group(path, P)
    Bd = _dev(B)
    Xd = torch.empty_like(Bd)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st, rep = solve_group(hs, Bd, Xd)
    err = rel_l2_cols(_host(Xd), ref.x)
    assert err.max() <= TOL, (P, nrhs, err.max())
    assert np.allclose(rep["it0"], ref.it0, rtol=1e-11)
    assert np.allclose(rep["it1"], ref.it1, rtol=1e-10)
    assert rep["n_diverged"] == int((ref.ratio >= 0.1).sum())
    # repeatable
    X2 = torch.empty_like(Bd)
    solve_group(hs, Bd, X2)
    assert torch.equal(X2, Xd)
    info = [h.info() for h in hs]
    for h in hs:
        h.close()
    return err, info


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("nrhs", [1, 70])
def test_group_c1(cfgdata, P, nrhs):
    _, info = _check(cfgdata("C1")["hm"], P, nrhs)
    assert info[0]["nranks"] == P
    assert info[0]["sep_rows"] > 0
    assert sum(i["own_rows"] for i in info) + info[0]["sep_rows"] == info[0]["N"]


@pytest.mark.parametrize("P", [2, 8])
def test_group_t2(cfgdata, P):
    _check(cfgdata("T2")["hm"], P, 5)


@pytest.mark.parametrize("kw", [dict(n_points=900, seed=7, clustered=True),
                                dict(n_points=2500, seed=5, leaf_edge=0.15)])
def test_group_synthetic(synthfile, kw):
    _check(synthfile(**kw)[0], 3, 9)


def test_group_c2_bench_size(cfgdata):
    """The bench config (C2, 181 RHS) split over 4 ranks."""
    meta = cfgdata("C2")
    from hmgen.build import read_rhs
    H = read_hm(meta["hm"])
    S = compute_scaling(H)
    B, _ = read_rhs(meta["rhs"])
    ref = solve(H, S, B)
    hs = _group(meta["hm"], 4)
    Bd = _dev(B)
    Xd = torch.empty_like(Bd)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        solve_group(hs, Bd, Xd)
    assert rel_l2_cols(_host(Xd), ref.x).max() <= TOL
    # every rank holds only its share of alpha panels, D^-1 and T (the far stacks stay whole),
    # and set up only its interior plus the separators (near blocks, W, panels, D^-1)
    h1 = PsHandle(meta["hm"], device=0)
    i1 = h1.info()
    h1.setup()
    whole = h1.info()["op_bytes"]
    h1.close()
    held = [h.info()["op_bytes"] for h in hs]
    assert max(held) < whole, (held, whole)
    sb = [h.info()["setup_bytes"] for h in hs]
    assert max(sb) < i1["setup_bytes"], (sb, i1["setup_bytes"])
    with pytest.raises(PsError) as e:          # per-operator diagnostics need the whole operator
        hs[0].apply(1, Bd, torch.empty_like(Bd))
    assert e.value.status == PS_ESTATE
    for h in hs:
        h.close()


def test_group_errors(cfgdata):
    path = cfgdata("C1")["hm"]
    hs = _group(path, 2)
    B = _dev(random_rhs(hs[0].N, 2, 0))
    X = torch.empty_like(B)
    with pytest.raises(PsError) as e:          # an in-process rank has no NCCL communicator
        hs[0].solve(B, X)
    assert e.value.status == PS_ESTATE
    h2 = PsHandle(path, device=0, rank=0, nranks=2, partition=True)
    with pytest.raises(PsError) as e:          # ... so its setup is the group's (ps_setup_group)
        h2.setup()
    assert e.value.status == PS_ESTATE
    h2.close()
    with pytest.raises(PsError) as e:          # ranks out of order
        solve_group([hs[1], hs[0]], B, X)
    assert e.value.status == PS_EINVAL
    for h in hs:
        h.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl_worker(rank, world, port, path, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2109_04129_b200 import nccl_unique_id
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        h = PsHandle(path, device=rank, rank=rank, nranks=world, partition=True, nccl_id=obj[0])
        h.setup()
        B = random_rhs(h.N, 4, 2)
        X = np.zeros_like(np.asfortranarray(B))
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            h.solve(np.asfortranarray(B), X)
        q.put((rank, X))
        h.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_nccl_two_ranks(cfgdata):
    import torch.multiprocessing as mp
    path = cfgdata("C1")["hm"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    H = read_hm(path)
    ref = solve(H, compute_scaling(H), random_rhs(H.N, 4, 2))
    for r in range(2):
        assert rel_l2_cols(out[r], ref.x).max() <= TOL
