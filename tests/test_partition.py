"""Row partition of the solve over ranks (SURVEY §8(e) option 1).

CPU tests (no GPU):
  * the partition libps computes (ps_partition, host-only) is a valid
    subtree-to-rank mapping of the elimination tree the oracle discovers
    (separators closed under struct, interior struct inside the rank's
    subtrees or the separators, far rows owned exactly once);
  * a world-size-2 gloo run of the partitioned phase schedule — each rank
    applies only its share of the operator (its interior alpha panels and
    D^-1, the replicated separators, its far rows) with the oracle's blocks,
    exchanging through torch.distributed exactly where libps does (sum
    all-reduce of separator rows after each interior forward sweep,
    all-gather of w and of x, all-reduce of the norm sums) — reproduces the
    oracle's single-process solve.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from tests.conftest import rel_l2_cols


def _part(path, P):
    from paper_2109_04129_b200 import partition
    return partition(path, P)


def _struct(S):
    return [sorted(S.alpha[k].keys()) for k in range(S.n)]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partition_invariants(cfgdata, synthfile, P):
    from oracle import compute_scaling, read_hm
    paths = [cfgdata("C1")["hm"], synthfile(n_points=900, seed=7, clustered=True)[0]]
    for path in paths:
        H = read_hm(path)
        S = compute_scaling(H)
        ow, fo = _part(path, P)
        st = _struct(S)
        assert len(ow) == S.n and len(fo) == S.n
        assert ow.min() >= -1 and ow.max() < P and fo.min() >= 0 and fo.max() < P
        if P == 1:
            assert (ow == 0).all() and (fo == 0).all()
            continue
        for k in range(S.n):
            if ow[k] < 0:
                assert all(ow[j] < 0 for j in st[k]), "separator struct must be separators"
            else:
                assert fo[k] == ow[k]
                assert all(ow[j] in (ow[k], -1) for j in st[k]), "interior struct leaves the subtree"
        # the split is real (a rank may stay empty when splitting further would
        # only move work into the replicated separators: C1 at P >= 4)
        assert len(set(ow[ow >= 0].tolist())) >= 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_model(H, S, ow, fo, g, b, dist, torch):
    """This rank's share of the partitioned two-term solve, exchanges via dist."""
    from oracle import apply_ZF
    o = S.offsets
    n = S.n
    mine = ow == g
    sep = ow < 0
    act = mine | sep

    def rows(mask):
        return np.concatenate([np.arange(o[k], o[k + 1]) for k in range(n) if mask[k]] or [np.zeros(0, int)])

    R_sep, R_mine = rows(sep), rows(mine)

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    def blk(v, k):
        return v[o[k]:o[k + 1]]

    def fwd(y, kset, src_mask):        # y_j += alpha_kj^T y_k for k in kset (elimination order)
        for k in range(n):
            if kset[k] and src_mask[k]:
                for j, a in S.alpha[k].items():
                    blk(y, j)[...] += a.T @ blk(y, k)

    def dinv(v):
        out = np.zeros_like(v)
        for k in range(n):
            if act[k]:
                blk(out, k)[...] = S.Dinv[k] @ blk(v, k)
        return out

    def bwd(v):
        w = np.zeros_like(v)
        for k in range(n - 1, -1, -1):
            if act[k]:
                acc = blk(v, k).copy()
                for j, a in S.alpha[k].items():
                    acc = acc + a @ blk(w, j)
                blk(w, k)[...] = acc
        return w

    def gather(v):                     # all-gather of the interior blocks (+ replicated separators)
        part = np.zeros_like(v)
        part[R_mine] = v[R_mine]
        full = allreduce(part)
        full[R_sep] = v[R_sep]
        return full

    # phase 0
    y = np.zeros_like(b)
    y[R_mine] = b[R_mine]
    if g == 0:
        y[R_sep] = b[R_sep]
    fwd(y, mine, mine)
    y[R_sep] = allreduce(y[R_sep])
    # phase 1
    fwd(y, sep, sep)
    bo = dinv(y)
    w = gather(bwd(bo))
    # phase 2: far rows of this rank, then the interior forward sweep of z
    t = apply_ZF(H, S, w)
    z = np.zeros_like(b)
    for k in range(n):
        if fo[k] == g:
            blk(z, k)[...] = blk(t, k)
    fwd(z, mine, mine)
    z[R_sep] = allreduce(z[R_sep])
    # phase 3
    fwd(z, sep, sep)
    xt = bo - dinv(z)
    nr = R_mine if g != 0 else np.concatenate([R_mine, R_sep])
    sums = allreduce(np.stack([(np.abs(bo[nr]) ** 2).sum(0), (np.abs((bo - xt)[nr]) ** 2).sum(0)]))
    x = gather(bwd(xt))
    return x, np.sqrt(sums)


def _worker(rank, world, port, path, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from hmgen.synth import random_rhs
        from oracle import compute_scaling, read_hm, solve
        H = read_hm(path)
        S = compute_scaling(H)
        ow, fo = _part(path, world)
        B = random_rhs(H.N, 3, 11)
        xe, norms = _rank_model(H, S, ow, fo, rank, B[S.e2rwg], dist, torch)
        if rank == 0:
            ref = solve(H, S, B)
            x = np.empty_like(xe)
            x[S.e2rwg] = xe
            q.put((float(rel_l2_cols(x, ref.x).max()),
                   float(np.abs(norms[0] - ref.it0).max() / ref.it0.max()),
                   float(np.abs(norms[1] - ref.it1).max() / ref.it1.max()),
                   int((ow < 0).sum())))
    finally:
        dist.destroy_process_group()


def test_row_partition_two_rank_gloo(synthfile):
    path, _ = synthfile(n_points=900, seed=7, clustered=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    err, e0, e1, nsep = q.get(timeout=10)
    assert nsep > 0                     # the exchange path is exercised
    assert err < 1e-12, err
    assert e0 < 1e-12 and e1 < 1e-12
