"""Sharded (multi-rank) logic on CPU: layout coverage, the deterministic
all-gather exchange over gloo (world size 2), and an end-to-end sharded
approximate product with the oracle standing in for the per-rank kernels."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_04940_b200.distributed import (ShardExchange, ShardLayout, exchange_sum, grid_shape,
                                                 pairwise_shards, shard_range, tree_combine)


def test_grid_and_ranges():
    assert [grid_shape(w) for w in (1, 2, 4, 8)] == [(1, 1), (1, 2), (2, 2), (2, 4)]
    for total, parts in [(10, 3), (16384, 8), (5, 8)]:
        pieces = [shard_range(total, parts, i) for i in range(parts)]
        assert pieces[0][0] == 0 and pieces[-1][1] == total
        assert all(a[1] == b[0] for a, b in zip(pieces, pieces[1:]))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_layout_reads_every_byte_once(world):
    m, n, p = 37, 3001, 1024
    tiles = np.zeros((m, p), int)
    cs_seen = np.zeros(n, int)
    rs_seen = np.zeros((n, p), int)
    for r in range(world):
        L = ShardLayout(world, r, m, n, p)
        a, b = L.coords
        tiles[L.rows[0]:L.rows[1], L.cols[0]:L.cols[1]] += 1
        if a == 0:  # every column slab's chain is carried once per row group
            c0, c1 = L.colsq_slab(b)
            cs_seen[c0:c1] += 1
        r0, r1 = L.rowsq_slab(a)
        rs_seen[r0:r1, L.cols[0]:L.cols[1]] += 1
    assert (tiles == 1).all() and (cs_seen == 1).all() and (rs_seen == 1).all()
    assert ShardLayout(world, 0, m, n, p).exact_rows


def test_pairwise_shards_are_tree_nodes():
    # the tree of numpy's pairwise sum over 1000 elements: 496 | 504, then 248 | 248 | 248 | 256
    assert pairwise_shards(1000, 2) == [(0, 496), (496, 1000)]
    assert pairwise_shards(1000, 4) == [(0, 248), (248, 496), (496, 744), (744, 1000)]
    assert pairwise_shards(200, 4) is None and pairwise_shards(1000, 3) is None
    g = np.random.default_rng(0)
    for p, parts in [(1000, 2), (1000, 4), (16384, 4), (777, 2), (4096, 8)]:
        x = g.standard_normal((5, p)) ** 2
        segs = pairwise_shards(p, parts)
        subs = [np.add.reduce(x[:, lo:hi], axis=1) for lo, hi in segs]
        assert np.array_equal(tree_combine(subs), np.add.reduce(x, axis=1)), (p, parts)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out_q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def _run(world, fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return [res[r] for r in range(world)]


def _exchange_fn(rank, world):
    part = torch.arange(5, dtype=torch.float64) * (rank + 1) + 0.1 * rank
    return exchange_sum(part).numpy()


def test_exchange_sum_gloo_world2():
    a, b = _run(2, _exchange_fn)
    expect = (torch.arange(5, dtype=torch.float64) * 1 + 0.0) + (torch.arange(5, dtype=torch.float64) * 2 + 0.1)
    assert np.array_equal(a, b) and np.array_equal(a, expect.numpy())


def _np_colsq(Mslab, acc, accumulate):
    """The per-rank colsq kernel restated in NumPy: the sequential chain, continued from acc."""
    sq = Mslab.numpy().astype(np.float64) ** 2
    if accumulate:
        sq = np.concatenate([acc.numpy()[None, :], sq], axis=0)
    acc.copy_(torch.from_numpy(np.add.reduce(sq, axis=0)))


def _np_rowsq(Nslab, out):
    out.copy_(torch.from_numpy(np.add.reduce(Nslab.numpy().astype(np.float64) ** 2, axis=1)))


def _sharded_fn(rank, world):
    """One rank of a sharded product with the NumPy restatement of the per-rank
    kernels: the exact exchange (chained colsq stages, tree-combined rowsq) and
    the plan/draws that follow, computed redundantly on every rank."""
    import workloads
    from oracle import blockmm_oracle as O
    M, N, sizes = workloads.cfg2(n=3000, m=40, p=1024, K=10)
    n = M.shape[1]
    L = ShardLayout(world, rank, M.shape[0], n, N.shape[1])
    ex = ShardExchange(L, colsq_fn=_np_colsq, rowsq_fn=_np_rowsq)
    a0, a1 = L.rows
    b0, b1 = L.cols
    cs, rs = torch.empty(n, dtype=torch.float64), torch.empty(n, dtype=torch.float64)
    ex.norms(torch.from_numpy(M[a0:a1].copy()), torch.from_numpy(N[:, b0:b1].copy()), cs, rs)
    cs, rs = cs.numpy(), rs.numpy()
    probs, s = O.block_stats(cs, rs, sizes)
    budgets, _ = O.plan_budgets("ONC", sizes, 600, s=s)
    streams = workloads.sample_rng(2, 7).spawn(len(sizes))
    cols, prob, scale, C, D = O.sketch(M[a0:a1], N[:, b0:b1], sizes, probs, budgets, streams)
    gpart = torch.from_numpy(O.block_product_sq(M[a0:a1], N[:, b0:b1], sizes))
    ex.sum_(gpart)
    return dict(colsq=cs, rowsq=rs, budgets=budgets, cols=cols, tile=(a0, a1, b0, b1), CD=C @ D, gsq=gpart.numpy())


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_product_gloo_matches_single(world):
    """World 2 (grid 1x2: tree-combined rowsq) and 4 (2x2: also two chained
    colsq stages): every rank holds the single-process norms BIT FOR BIT, so the
    budgets and draws equal the oracle's on one device; the tiles assemble C.D
    and the exchanged g_k^2 partials sum to the oracle's."""
    import workloads
    from oracle import blockmm_oracle as O
    res = _run(world, _sharded_fn)
    M, N, sizes = workloads.cfg2(n=3000, m=40, p=1024, K=10)
    assert np.array_equal(res[0]["colsq"], O.colsq(M)) and np.array_equal(res[0]["rowsq"], O.rowsq(N))
    ref = O.approx_product(M, N, sizes, 600, "ONC", workloads.sample_rng(2, 7))
    CD = np.zeros_like(ref["CD"])
    for r in res:
        assert np.array_equal(r["colsq"], res[0]["colsq"]) and np.array_equal(r["rowsq"], res[0]["rowsq"])
        assert np.array_equal(r["budgets"], ref["budgets"])
        assert np.array_equal(r["cols"], ref["columns"])
        assert np.array_equal(r["gsq"], res[0]["gsq"])
        a0, a1, b0, b1 = r["tile"]
        CD[a0:a1, b0:b1] = r["CD"]
    assert np.linalg.norm(CD - ref["CD"]) / np.linalg.norm(ref["CD"]) < 1e-12
    gsq = O.block_product_sq(M, N, sizes)
    assert np.allclose(res[0]["gsq"], gsq, rtol=1e-12, atol=0)
