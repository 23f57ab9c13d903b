"""World-size-2 gloo test of the multi-process (N > 1) host path on CPU.

Two processes split the RHS block with paper_2109_04129_b200.dist, solve their
columns (the oracle stands in for the GPU solve on CPU), take the max of their
timings and gather the columns; rank 0 checks the gathered solution equals a
single-process solve column for column.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, path, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from hmgen.synth import random_rhs
        from oracle import compute_scaling, read_hm, solve
        from paper_2109_04129_b200.dist import column_slice, gather_columns, max_over_ranks
        H = read_hm(path)
        S = compute_scaling(H)
        nrhs = 7
        B = random_rhs(H.N, nrhs, 5)
        sl = column_slice(nrhs, world, rank, "strong")
        X = solve(H, S, B[:, sl]).x
        t = max_over_ranks(10.0 + rank, dist)
        Xg = gather_columns(X, nrhs, dist, "strong")
        if rank == 0:
            ref = solve(H, S, B).x
            q.put((float(np.abs(Xg - ref).max() / np.abs(ref).max()), t,
                   [column_slice(nrhs, world, r, "strong") for r in range(world)]))
    finally:
        dist.destroy_process_group()


def test_column_slices():
    from paper_2109_04129_b200.dist import column_slice
    for n in (1, 7, 181):
        for w in (1, 2, 4, 8):
            sl = [column_slice(n, w, r, "strong") for r in range(w)]
            cover = np.concatenate([np.arange(n)[s] for s in sl])
            assert np.array_equal(cover, np.arange(n))
            assert max(s.stop - s.start for s in sl) - min(s.stop - s.start for s in sl) <= 1
            assert all(column_slice(n, w, r, "weak") == slice(0, n) for r in range(w))


def test_two_rank_gloo(synthfile):
    path, _ = synthfile(n_points=300, seed=21)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs)
    err, t, slices = q.get(timeout=10)
    assert err < 1e-14                 # columns are independent: bitwise-equal up to BLAS order
    assert t == 11.0                   # max over ranks
    assert slices == [slice(0, 4), slice(4, 7)]
