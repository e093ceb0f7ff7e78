"""K7 in Gram form (bmm_segsq_gram): OPL block-product norms
g_k^2 = ||M^k N_k||_F^2 = <M^k^T M^k, N_k N_k^T> against the oracle's
multiplied-out blocks (block_scores, plan.py:176-189), and the OPL pipeline on
this engine bit-exact in budgets and draws; the batched / float32 SSM pipeline
(estimators.py:221-253) against the oracle."""
import numpy as np
import pytest

import workloads
from oracle import blockmm_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
bm = pytest.importorskip("paper_2105_04940_b200")
from paper_2105_04940_b200 import _lib  # noqa: E402
from paper_2105_04940_b200.pipeline import SketchPipeline, seeds_from_rngs  # noqa: E402


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def gram(M, N, sizes, batch=1):
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    K = len(sizes)
    off = torch.as_tensor(O.offsets_of(sizes), device="cuda")
    out = torch.full((batch * K,), -1.0, dtype=torch.float64, device="cuda")
    m, n = Md.shape[-2:]
    p = Nd.shape[-1]
    _lib.call("bmm_segsq_gram", _lib.matrix_dtype(Md), Md.data_ptr(), Md.stride(-2), m * n if batch > 1 else 0,
              Nd.data_ptr(), Nd.stride(-2), n * p if batch > 1 else 0, m, p, off.data_ptr(), K, 0, batch,
              out.data_ptr(), _lib.stream_ptr())
    return out.view(batch, K).cpu().numpy()


def check_gsq(got, M, N, sizes):
    ref = O.block_product_sq(M.astype(np.float64), N.astype(np.float64), sizes)
    cs, rs = O.colsq(M.astype(np.float64)), O.rowsq(N.astype(np.float64))
    _, s = O.block_stats(cs, rs, sizes)
    # relative to g^2 where it is not tiny against s^2 (the radicand's scale)
    err = np.abs(got - ref)
    assert (err <= 1e-12 * np.maximum(ref, 1e-3 * s ** 2)).all(), (err / np.maximum(ref, 1e-300)).max()
    return ref


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("shape", [(40, 30, (64, 64, 1, 7, 33, 64, 17)), (300, 257, (64,) * 8),
                                   (1, 5, (3, 64, 2)), (129, 1, (16, 48))])
def test_gram_matches_multiplied_blocks(dtype, shape):
    m, p, sizes = shape
    g = np.random.default_rng(17)
    n = sum(sizes)
    M = (g.standard_normal((m, n)) * g.lognormal(0, 1, n)).astype(dtype)
    N = (g.standard_normal((n, p)) * g.lognormal(0, 1, n)[:, None]).astype(dtype)
    got = gram(M, N, sizes)[0]
    check_gsq(got, M, N, sizes)


def test_gram_zero_block_and_batch():
    g = np.random.default_rng(3)
    sizes = (64, 20, 64, 5)
    n = sum(sizes)
    B = 3
    M = g.standard_normal((B, 70, n))
    N = g.standard_normal((B, n, 90))
    M[1, :, 64:84] = 0.0  # block 1 of problem 1: M^k = 0 -> g = 0 exactly
    got = gram(M, N, sizes, batch=B)
    for b in range(B):
        check_gsq(got[b], M[b], N[b], sizes)
    assert got[1, 1] == 0.0


def test_gram_unaligned_rows():
    """Odd leading dimensions and block starts: the per-element copy path."""
    g = np.random.default_rng(5)
    sizes = (13, 50, 7, 1, 60)
    n = sum(sizes)
    N = g.standard_normal((n, 41))
    # M is a column window of a wider matrix: odd leading dimension, unaligned rows
    Md = torch.as_tensor(np.ascontiguousarray(g.standard_normal((33, n + 3))), device="cuda")[:, 1:n + 1]
    M = Md.cpu().numpy()
    off = torch.as_tensor(O.offsets_of(sizes), device="cuda")
    Nd = torch.as_tensor(N, device="cuda")
    out = torch.empty(len(sizes), dtype=torch.float64, device="cuda")
    _lib.call("bmm_segsq_gram", _lib.BMM_F64, Md.data_ptr(), Md.stride(0), 0, Nd.data_ptr(), Nd.stride(0), 0,
              33, 41, off.data_ptr(), len(sizes), 0, 1, out.data_ptr(), _lib.stream_ptr())
    check_gsq(out.cpu().numpy(), M, N, sizes)


def test_engine_choice():
    from paper_2105_04940_b200.plan import segsq_engine
    assert segsq_engine(64, 16384, 16384, 262144) == "gram"   # config 4
    assert segsq_engine(64, 256, 256, 4096) == "gram"         # config 5
    assert segsq_engine(1000, 500, 500, 20000) in ("i8", "dmma")  # config 2: long blocks
    assert segsq_engine(100, 200, 200, 10000) == "dmma"       # config 1: > 64 columns


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_opl_pipeline_on_gram_engine(dtype):
    """Config-5 shaped OPL problems (256 x 4096 . 4096 x 256, K=64 x 64): the
    pipeline's g_k^2 from the Gram kernel gives the oracle's budgets and draws."""
    B, m, n, p, K, W = 4, 256, 4096, 256, 64, 1024
    probs = [workloads.cfg5_problem(b) for b in range(B)]
    Ms = np.stack([x[0] for x in probs]).astype(dtype)
    Ns = np.stack([x[1] for x in probs]).astype(dtype)
    Md, Nd = torch.as_tensor(Ms, device="cuda"), torch.as_tensor(Ns, device="cuda")
    sizes = (64,) * K
    pipe = SketchPipeline(m, n, p, sizes, W, "OPL", batch=B, dtype=Md.dtype)
    assert pipe.seg_engine == "gram"
    CD = pipe.run(Md, Nd, seeds_from_rngs("OPL", [workloads.sample_rng(5, b) for b in range(B)], K)).cpu().numpy()
    pipe.check()
    tol = 1e-12 if dtype == np.float64 else 1e-5
    for b in range(B):
        M64, N64 = Ms[b].astype(np.float64), Ns[b].astype(np.float64)
        ref = O.approx_product(M64, N64, sizes, W, "OPL", workloads.sample_rng(5, b))
        g = pipe.gsq.view(B, K)[b].cpu().numpy()
        assert np.abs(g - ref["gsq"]).max() <= 1e-12 * ref["gsq"].max()
        assert np.array_equal(pipe.budgets_host()[b], ref["budgets"]), b
        assert np.array_equal(pipe.columns_host()[b], ref["columns"]), b
        assert np.array_equal(pipe.scales_host()[b], ref["scale"]), b
        assert rel(CD[b], ref["CD"]) < tol


def test_allocate_optimal_api_on_gram_engine(monkeypatch):
    monkeypatch.setenv("BMM_SEGSQ", "gram")
    M, N = workloads.cfg5_problem(3)
    M, N = M.astype(np.float64), N.astype(np.float64)
    sizes = (64,) * 64
    plan = bm.allocate_optimal(M, N, bm.BlockPartition(sizes), 1024)
    cs, rs, probs, s = O.instance_stats(M, N, sizes)
    ref, _ = O.plan_budgets("OPL", sizes, 1024, s=s, aux_sq=O.block_product_sq(M, N, sizes))
    assert np.array_equal(plan.budgets, ref)
    sc = bm.block_scores(M, N, bm.BlockPartition(sizes))
    assert np.allclose(sc.product_norms ** 2, O.block_product_sq(M, N, sizes), rtol=1e-12, atol=0)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("graph", [False, True])
def test_ssm_pipeline_batched(dtype, graph):
    """Batched SSM (whole-block draws from each problem's caller stream) through
    the compressed gather and the float64 DMMA / float32 tcgen05 contraction."""
    B, m, n, p, K, draws = 5, 96, 2048, 80, 32, 12
    g = np.random.default_rng(11)
    Ms = (g.standard_normal((B, m, n)) * g.lognormal(0, 1, (B, 1, n))).astype(dtype)
    Ns = (g.standard_normal((B, n, p)) * g.lognormal(0, 1, (B, n, 1))).astype(dtype)
    Md, Nd = torch.as_tensor(Ms, device="cuda"), torch.as_tensor(Ns, device="cuda")
    sizes = (n // K,) * K
    pipe = SketchPipeline(m, n, p, sizes, 0, "SSM", batch=B, dtype=Md.dtype, draws=draws)
    if graph:
        pipe.run(Md, Nd, seeds_from_rngs("SSM", [np.random.default_rng(0) for _ in range(B)], K, draws))
        pipe.capture(Md, Nd)
    rngs = [np.random.default_rng(100 + b) for b in range(B)]
    CD = pipe.run(Md, Nd, seeds_from_rngs("SSM", rngs, K, draws)).cpu().numpy()
    pipe.check()
    tol = 1e-12 if dtype == np.float64 else 1e-5
    for b in range(B):
        ref_rng = np.random.default_rng(100 + b)
        ref = O.ssm_product(Ms[b].astype(np.float64), Ns[b].astype(np.float64), sizes, draws, ref_rng)
        assert np.array_equal(pipe.columns_host()[b], ref["blocks"]), b
        assert np.allclose(pipe.scales_host()[b], ref["scale"], rtol=1e-13, atol=0), b
        assert rel(CD[b], ref["CD"]) < tol
        # the caller's generator is left where the reference leaves it
        assert rngs[b].random() == ref_rng.random()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("m,p,sizes,batch", [(300, 128, (64,) * 10, 1), (129, 1024, (1, 63, 64, 17, 40), 1),
                                             (64, 16384, (64,) * 3, 1), (100, 256, (32,) * 8, 3)])
def test_gram_norms_fused_bit_exact(dtype, m, p, sizes, batch):
    """bmm_segsq_gram_norms: g_k^2 as bmm_segsq_gram, and the norm pass riding in
    the same read of M and N -- colsq (sequential over the rows) and rowsq
    (NumPy's pairwise tree, p = 128 * 2^k) bit-identical to the oracle's NumPy
    order; ragged segments, rows not a multiple of the 32-row stage, batches."""
    g = np.random.default_rng(m + p + len(sizes))
    n = sum(sizes)
    M = (g.standard_normal((batch, m, n)) * g.lognormal(0, 2, (batch, 1, n))).astype(dtype)
    N = (g.standard_normal((batch, n, p)) * g.lognormal(0, 2, (batch, n, 1))).astype(dtype)
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    K = len(sizes)
    off = torch.as_tensor(O.offsets_of(sizes), device="cuda")
    gsq = torch.full((batch * K,), -1.0, dtype=torch.float64, device="cuda")
    cs = torch.full((batch * n,), -1.0, dtype=torch.float64, device="cuda")
    rs = torch.full((batch * n,), -1.0, dtype=torch.float64, device="cuda")
    _lib.call("bmm_segsq_gram_norms", _lib.matrix_dtype(Md), Md.data_ptr(), n, m * n, Nd.data_ptr(), p, n * p, m, p,
              off.data_ptr(), K, 0, batch, gsq.data_ptr(), cs.data_ptr(), rs.data_ptr(), n, _lib.stream_ptr())
    ref = gram(M if batch > 1 else M[0], N if batch > 1 else N[0], sizes, batch)
    assert np.array_equal(gsq.view(batch, K).cpu().numpy(), ref)  # the Gram part: the unfused kernel's bits
    for b in range(batch):
        M64, N64 = M[b].astype(np.float64), N[b].astype(np.float64)
        assert np.array_equal(cs[b * n:(b + 1) * n].cpu().numpy(), O.colsq(M64)), b
        assert np.array_equal(rs[b * n:(b + 1) * n].cpu().numpy(), O.rowsq(N64)), b
    with pytest.raises(RuntimeError, match="128"):
        _lib.call("bmm_segsq_gram_norms", _lib.matrix_dtype(Md), Md.data_ptr(), n, m * n, Nd.data_ptr(), p, n * p,
                  m, p - 1, off.data_ptr(), K, 0, batch, gsq.data_ptr(), cs.data_ptr(), rs.data_ptr(), n,
                  _lib.stream_ptr())


@pytest.mark.parametrize("fused", ["0", "1"])
def test_opl_group_with_fused_stats(fused, monkeypatch):
    """The config-4 step's shared statistics with the norm pass fused into the
    Gram kernel (opt-in, BMM_FUSED_STATS=1) or separate: identical budgets,
    draws and products."""
    from paper_2105_04940_b200.pipeline import PipelineGroup
    monkeypatch.setenv("BMM_FUSED_STATS", fused)
    g = np.random.default_rng(5)
    sizes = (64,) * 32
    n = sum(sizes)
    M = (g.standard_normal((200, n)) * np.repeat(g.uniform(0.1, 10, 32), 64)).astype(np.float32)
    N = (g.standard_normal((n, 256)) * np.repeat(g.uniform(0.1, 10, 32), 64)[:, None]).astype(np.float32)
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    group = PipelineGroup([SketchPipeline(200, n, 256, sizes, 512, "OPL", dtype=torch.float32),
                           SketchPipeline(200, n, 256, sizes, 512, "ONC", dtype=torch.float32)])
    assert group.shared.fused(Md) == (fused == "1")
    group.run(Md, Nd, [seeds_from_rngs("OPL", [np.random.default_rng(1)], 32),
                       seeds_from_rngs("ONC", [np.random.default_rng(2)], 32)])
    group.capture(Md, Nd)
    for s in (3, 4):
        sd = [seeds_from_rngs("OPL", [np.random.default_rng(s)], 32),
              seeds_from_rngs("ONC", [np.random.default_rng(s + 9)], 32)]
        outs = [o.cpu().numpy() for o in group.run(Md, Nd, sd)]
        group.check()
        M64, N64 = M.astype(np.float64), N.astype(np.float64)
        assert np.array_equal(group.shared.colsq.cpu().numpy(), O.colsq(M64))
        assert np.array_equal(group.shared.rowsq.cpu().numpy(), O.rowsq(N64))
        for i, meth in enumerate(("OPL", "ONC")):
            ref = O.approx_product(M64, N64, sizes, 512, meth, np.random.default_rng(s + 9 * i))
            assert np.array_equal(group.pipes[i].budgets_host()[0], ref["budgets"]), meth
            assert np.array_equal(group.pipes[i].columns_host()[0], ref["columns"]), meth
            assert rel(outs[i], ref["CD"]) < 1e-5, meth
