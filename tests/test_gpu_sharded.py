"""The sharded product (distributed.ShardedApproxProduct) at world 2 (grid 1x2)
and 4 (2x2) as separate processes on one B200 with a gloo group (host-staged
exchange: no rank's kernel waits on another's).  Every rank's norms are the
single-GPU bits (chained colsq stages, tree-combined rowsq), so budgets and
draws of OPL, ONC, ONU and SSM equal the single-GPU PipelineGroup's and the
oracle's; the assembled tiles equal its products within the dtype's bar."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

RUNS = [("OPL", 2048), ("ONC", 2048), ("ONU", 2048), ("SSM", 24)]


def _instance(dtype):
    g = np.random.default_rng(21)
    sizes = (64,) * 128
    n = sum(sizes)
    M = (g.standard_normal((384, n)) * np.repeat(g.uniform(0.1, 10, 128), 64)).astype(dtype)
    N = (g.standard_normal((n, 1024)) * np.repeat(g.uniform(0.1, 10, 128), 64)[:, None]).astype(dtype)
    return M, N, sizes


def _seeds(K):
    from paper_2105_04940_b200.pipeline import seeds_from_rngs
    return [seeds_from_rngs(m, [np.random.default_rng(100 + i)], K, draws=c) for i, (m, c) in enumerate(RUNS)]


def _rank(rank, world, port, dtype, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2105_04940_b200.distributed import ShardLayout, ShardedApproxProduct
        M, N, sizes = _instance(dtype)
        L = ShardLayout(world, rank, M.shape[0], M.shape[1], N.shape[1])
        (a0, a1), (b0, b1) = L.rows, L.cols
        tdt = torch.float64 if dtype == np.float64 else torch.float32
        sh = ShardedApproxProduct(L, sizes, RUNS, dtype=tdt, c0=256)
        Ml = torch.as_tensor(M[a0:a1], device="cuda")
        Nl = torch.as_tensor(np.ascontiguousarray(N[:, b0:b1]), device="cuda")
        tiles = [t.cpu().numpy() for t in sh.run(Ml, Nl, _seeds(len(sizes)))]
        sh.check()
        out = dict(tile=(a0, a1, b0, b1), tiles=tiles, cols=[p.columns_host()[0] for p in sh.pipes],
                   budgets=[p.budgets_host()[0] for p in sh.pipes if p.method != "SSM"],
                   colsq=sh.pipes[0].colsq.cpu().numpy(), rowsq=sh.pipes[0].rowsq.cpu().numpy())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _spawn(world, dtype):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_rank, args=(r, world, port, dtype, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return [res[r] for r in range(world)]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_sharded_world_matches_single_gpu(world, dtype):
    from oracle import blockmm_oracle as O
    from paper_2105_04940_b200.pipeline import PipelineGroup, SketchPipeline
    M, N, sizes = _instance(dtype)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    m, n, p = M.shape[0], M.shape[1], N.shape[1]
    grp = PipelineGroup([SketchPipeline(m, n, p, sizes, 0, "SSM", draws=c, dtype=tdt) if meth == "SSM" else
                         SketchPipeline(m, n, p, sizes, c, meth, c0=256, dtype=tdt) for meth, c in RUNS])
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    want = [o.cpu().numpy() for o in grp.run(Md, Nd, _seeds(len(sizes)))]
    grp.check()
    res = _spawn(world, dtype)
    M64, N64 = M.astype(np.float64), N.astype(np.float64)
    cs, rs = O.colsq(M64), O.rowsq(N64)
    tol = 1e-12 if dtype == np.float64 else 1e-5
    for i, (meth, c) in enumerate(RUNS):
        CD = np.zeros((m, p), dtype=want[i].dtype)
        for r in res:
            assert np.array_equal(r["colsq"], cs) and np.array_equal(r["rowsq"], rs)
            assert np.array_equal(r["cols"][i], grp.pipes[i].columns_host()[0]), (meth, "draws")
            a0, a1, b0, b1 = r["tile"]
            CD[a0:a1, b0:b1] = r["tiles"][i]
        assert np.linalg.norm(CD - want[i]) / np.linalg.norm(want[i]) < tol, meth
    for r in res:
        for j, pipe in enumerate([q for q in grp.pipes if q.method != "SSM"]):
            assert np.array_equal(r["budgets"][j], pipe.budgets_host()[0])


def test_nccl_comm_exchanges_world1(monkeypatch):
    """The C-ABI NCCL exchanges (bmm_nccl_comm_init, bmm_all_gather_f64_nccl,
    bmm_exchange_sum_nccl) on a one-rank communicator -- this box has one GPU,
    and NCCL refuses two ranks on one device -- and the sharded product run
    through them (the collective runs even at world 1) against the single-GPU
    PipelineGroup, bit for bit."""
    from paper_2105_04940_b200 import _lib
    from paper_2105_04940_b200.distributed import NcclComm, ShardLayout, ShardedApproxProduct
    from paper_2105_04940_b200.pipeline import PipelineGroup, SketchPipeline
    assert _lib.load().bmm_nccl_version() >= 22000
    comm = NcclComm()
    x = torch.randn(1000, dtype=torch.float64, device="cuda")
    g = comm.all_gather(x)
    assert g.shape == (1, 1000) and torch.equal(g[0], x)
    assert torch.equal(comm.exchange_sum(x), x)
    M, N, sizes = _instance(np.float32)
    m, n, p = M.shape[0], M.shape[1], N.shape[1]
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    grp = PipelineGroup([SketchPipeline(m, n, p, sizes, 0, "SSM", draws=c, dtype=torch.float32) if meth == "SSM" else
                         SketchPipeline(m, n, p, sizes, c, meth, c0=256, dtype=torch.float32) for meth, c in RUNS])
    want = [o.cpu().numpy() for o in grp.run(Md, Nd, _seeds(len(sizes)))]
    monkeypatch.setenv("BMM_EXCHANGE_WORLD1", "1")
    sh = ShardedApproxProduct(ShardLayout(1, 0, m, n, p), sizes, RUNS, dtype=torch.float32, c0=256, comm=comm)
    got = [t.cpu().numpy() for t in sh.run(Md, Nd, _seeds(len(sizes)))]
    sh.check()
    for i, (meth, _) in enumerate(RUNS):
        assert np.array_equal(sh.pipes[i].columns_host(), grp.pipes[i].columns_host()), meth
        assert np.array_equal(got[i], want[i]), meth
    comm.close()
