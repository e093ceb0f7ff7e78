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

from paper_2105_04940_b200.distributed import ShardLayout, exchange_sum, grid_shape, shard_range


def test_grid_and_ranges():
    assert [grid_shape(w) for w in (1, 2, 4, 8)] == [(1, 1), (1, 2), (2, 2), (2, 4)]
    for total, parts in [(10, 3), (16384, 8), (5, 8)]:
        pieces = [shard_range(total, parts, i) for i in range(parts)]
        assert pieces[0][0] == 0 and pieces[-1][1] == total
        assert all(a[1] == b[0] for a, b in zip(pieces, pieces[1:]))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_layout_reads_every_byte_once(world):
    m, n, p = 37, 11, 29
    rows_seen = np.zeros(m, int)
    cols_seen = np.zeros(p, int)
    tiles = np.zeros((m, p), int)
    for r in range(world):
        L = ShardLayout(world, r, m, n, p)
        a0, a1 = L.norm_rows
        b0, b1 = L.norm_cols
        rows_seen[a0:a1] += 1
        cols_seen[b0:b1] += 1
        assert L.rows[0] <= a0 <= a1 <= L.rows[1] and L.cols[0] <= b0 <= b1 <= L.cols[1]
        tiles[L.rows[0]:L.rows[1], L.cols[0]:L.cols[1]] += 1
    assert (rows_seen == 1).all() and (cols_seen == 1).all() and (tiles == 1).all()


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
    res = dict(q.get(timeout=300) for _ in procs)
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


def _sharded_fn(rank, world):
    """Per-rank work of ShardedApproxProduct, with oracle NumPy in place of the kernels."""
    import workloads
    from oracle import blockmm_oracle as O
    M, N, sizes = workloads.cfg2(n=3000, m=40, p=36, K=10)
    L = ShardLayout(world, rank, M.shape[0], M.shape[1], N.shape[1])
    r0, r1 = L.norm_rows
    c0, c1 = L.norm_cols
    n = M.shape[1]
    part = np.zeros(2 * n)
    part[:n] = O.colsq(M[r0:r1]) if r1 > r0 else 0.0
    part[n:] = O.rowsq(N[:, c0:c1]) if c1 > c0 else 0.0
    full = exchange_sum(torch.as_tensor(part)).numpy()
    probs, s = O.block_stats(full[:n], full[n:], sizes)
    budgets, _ = O.plan_budgets("ONC", sizes, 600, s=s)
    streams = workloads.sample_rng(2, 7).spawn(len(sizes))
    a0, a1 = L.rows
    b0, b1 = L.cols
    cols, prob, scale, C, D = O.sketch(M[a0:a1], N[:, b0:b1], sizes, probs, budgets, streams)
    return dict(budgets=budgets, cols=cols, tile=(a0, a1, b0, b1), CD=C @ D)


def test_sharded_product_gloo_world2_matches_single():
    import workloads
    from oracle import blockmm_oracle as O
    res = _run(2, _sharded_fn)
    # identical plan and draws on every rank (no broadcast needed)
    assert np.array_equal(res[0]["budgets"], res[1]["budgets"])
    assert np.array_equal(res[0]["cols"], res[1]["cols"])
    M, N, sizes = workloads.cfg2(n=3000, m=40, p=36, K=10)
    ref = O.approx_product(M, N, sizes, 600, "ONC", workloads.sample_rng(2, 7))
    assert np.array_equal(res[0]["budgets"], ref["budgets"])
    assert np.array_equal(res[0]["cols"], ref["columns"])
    CD = np.zeros_like(ref["CD"])
    for r in res:
        a0, a1, b0, b1 = r["tile"]
        CD[a0:a1, b0:b1] = r["CD"]
    assert np.linalg.norm(CD - ref["CD"]) / np.linalg.norm(ref["CD"]) < 1e-12
