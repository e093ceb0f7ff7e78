"""The device-resident pipeline (paper_2105_04940_b200.pipeline) is bit-identical
to the per-call API and to the oracle, eagerly, under CUDA-graph replay and
batched over problems."""
import numpy as np
import pytest

import workloads
from oracle import blockmm_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
bm = pytest.importorskip("paper_2105_04940_b200")
from paper_2105_04940_b200.pipeline import PipelineGroup, SketchPipeline, seeds_from_rngs  # noqa: E402


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


@pytest.mark.parametrize("method", ["OPL", "ONC", "UU", "ONU", "ONMCNR"])
@pytest.mark.parametrize("graph", [False, True])
def test_pipeline_matches_oracle(method, graph):
    M, N, sizes = workloads.cfg2(n=4000, m=60, p=50, K=12)
    c, c0 = 300, 120
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    pipe = SketchPipeline(60, 4000, 50, sizes, c, method, c0=c0)
    if graph:
        pipe.run(Md, Nd, seeds_from_rngs(method, [np.random.default_rng(1)], len(sizes)))
        pipe.capture(Md, Nd)
    for seed in (5, 6):
        rng = np.random.default_rng(seed)
        CD = pipe.run(Md, Nd, seeds_from_rngs(method, [rng], len(sizes))).cpu().numpy()
        pipe.check()
        ref = O.approx_product(M, N, sizes, c, method, np.random.default_rng(seed), c0=c0)
        assert np.array_equal(pipe.budgets_host()[0], ref["budgets"]), method
        assert np.array_equal(pipe.columns_host()[0], ref["columns"]), method
        assert np.array_equal(pipe.scales_host()[0], ref["scale"]), method
        assert rel(CD, ref["CD"]) < 1e-12


@pytest.mark.parametrize("shared", [False, True])
def test_pipeline_group_concurrent_replay_is_bit_identical(shared):
    """A c x method sweep replayed as one graph with concurrent branches gives
    exactly the products of the member pipelines run one by one -- also when the
    members share one statistics stage (norms, probabilities, g_k once)."""
    M, N, sizes = workloads.cfg2(n=4000, m=60, p=50, K=12)
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    runs = [(c, meth) for c in (200, 400) for meth in ("OPL", "ONC", "ONMCNR", "UU", "ONU")]
    solo = [SketchPipeline(60, 4000, 50, sizes, c, meth, c0=120) for c, meth in runs]
    group = PipelineGroup([SketchPipeline(60, 4000, 50, sizes, c, meth, c0=120) for c, meth in runs], joint=False,
                          shared=shared)
    assert (group.shared is not None) == shared
    seeds = lambda s: [seeds_from_rngs(meth, [np.random.default_rng(s + i)], len(sizes))  # noqa: E731
                       for i, (c, meth) in enumerate(runs)]
    eager = [o.clone() for o in group.run(Md, Nd, seeds(10))]
    group.capture(Md, Nd)
    assert group.graph_launches > 0
    for s in (10, 20):
        outs = [o.clone() for o in group.run(Md, Nd, seeds(s))]
        group.check()
        for i, pipe in enumerate(solo):
            ref = pipe.run(Md, Nd, seeds(s)[i])
            assert torch.equal(outs[i], ref), runs[i]
            assert np.array_equal(group.pipes[i].columns_host(), pipe.columns_host())
            if s == 10:
                assert torch.equal(eager[i], ref), runs[i]
    if shared:
        with pytest.raises(RuntimeError):
            group.pipes[1].run(Md, Nd, seeds(3)[1])


@pytest.mark.parametrize("serial,fork", [("0", "1"), ("1", "1"), ("0", "0")])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_shared_stats_group_with_ssm_matches_oracle(dtype, serial, fork, monkeypatch):
    """OPL, ONC and SSM over one instance with one shared statistics stage (the
    config-4 step): budgets, draws and scales bit-exact to the oracle, products
    within the dtype's bar, eager and replayed -- with g_k^2 forked beside the
    norm pass or after it (BMM_GSQ_FORK), and after the instance changes in
    place between replays (every statistic recomputed, none stale)."""
    g = np.random.default_rng(44)
    sizes = (64,) * 40
    n = sum(sizes)
    M = (g.standard_normal((96, n)) * np.repeat(g.uniform(0.1, 10, 40), 64)).astype(dtype)
    N = (g.standard_normal((n, 80)) * np.repeat(g.uniform(0.1, 10, 40), 64)[:, None]).astype(dtype)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    W, draws = 640, 10
    monkeypatch.setenv("BMM_GROUP_SERIAL", serial)  # members as concurrent branches, or one after another
    monkeypatch.setenv("BMM_GSQ_FORK", fork)
    group = PipelineGroup([SketchPipeline(96, n, 80, sizes, W, "OPL", dtype=tdt),
                           SketchPipeline(96, n, 80, sizes, W, "ONC", dtype=tdt),
                           SketchPipeline(96, n, 80, sizes, 0, "SSM", draws=draws, dtype=tdt)])
    assert group.shared is not None and group.shared.needs_gsq
    tol = 1e-12 if dtype == np.float64 else 1e-5
    M64, N64 = M.astype(np.float64), N.astype(np.float64)
    for rep, s in enumerate((5, 6, 7)):
        if rep == 1:
            group.capture(Md, Nd)
        if rep == 2:  # new data in the captured buffers: block 0 and 7 of M rescaled
            for k, f in ((0, 3.0), (7, 0.25)):
                M[:, 64 * k:64 * (k + 1)] = (M[:, 64 * k:64 * (k + 1)] * f).astype(dtype)
            Md.copy_(torch.as_tensor(M, device="cuda"))
            M64 = M.astype(np.float64)
        rngs = [np.random.default_rng(s + i) for i in range(3)]
        sd = [seeds_from_rngs("OPL", [rngs[0]], 40), seeds_from_rngs("ONC", [rngs[1]], 40),
              seeds_from_rngs("SSM", [rngs[2]], 40, draws=draws)]
        outs = [o.cpu().numpy() for o in group.run(Md, Nd, sd)]
        group.check()
        for i, meth in enumerate(("OPL", "ONC")):
            ref = O.approx_product(M64, N64, sizes, W, meth, np.random.default_rng(s + i))
            assert np.array_equal(group.pipes[i].budgets_host()[0], ref["budgets"]), meth
            assert np.array_equal(group.pipes[i].columns_host()[0], ref["columns"]), meth
            assert np.array_equal(group.pipes[i].scales_host()[0], ref["scale"]), meth
            assert rel(outs[i], ref["CD"]) < tol, meth
        ref = O.ssm_product(M64, N64, sizes, draws, np.random.default_rng(s + 2))
        assert np.array_equal(group.pipes[2].columns_host()[0], ref["blocks"])
        np.testing.assert_allclose(group.pipes[2].scales_host()[0], ref["scale"], rtol=1e-13)
        assert rel(outs[2], ref["CD"]) < tol


@pytest.mark.parametrize("m,p", [(60, 50), (200, 130)])
def test_pipeline_group_joint_gemm(m, p):
    """Joint mode: the members gather into pooled operands and ONE batched GEMM
    contracts them all.  Draws, budgets and scales are bit-identical to solo runs,
    products agree to 1e-13 (only the split of the inner sum differs) and match the
    oracle to 1e-12, eagerly and replayed; a member cannot be run on its own."""
    M, N, sizes = workloads.cfg2(n=4000, m=m, p=p, K=12)
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    runs = [(c, meth) for c in (200, 400, 900) for meth in ("OPL", "ONC", "ONMCNR")]
    solo = [SketchPipeline(m, 4000, p, sizes, c, meth, c0=120) for c, meth in runs]
    group = PipelineGroup([SketchPipeline(m, 4000, p, sizes, c, meth, c0=120) for c, meth in runs])
    assert group.joint
    seeds = lambda s: [seeds_from_rngs(meth, [np.random.default_rng(s + i)], len(sizes))  # noqa: E731
                       for i, (c, meth) in enumerate(runs)]
    eager = [o.clone() for o in group.run(Md, Nd, seeds(3))]
    group.capture(Md, Nd)
    for s in (3, 11):
        outs = [o.clone() for o in group.run(Md, Nd, seeds(s))]
        group.check()
        for i, pipe in enumerate(solo):
            ref = pipe.run(Md, Nd, seeds(s)[i])
            assert np.array_equal(group.pipes[i].columns_host(), pipe.columns_host()), runs[i]
            assert np.array_equal(group.pipes[i].scales_host(), pipe.scales_host()), runs[i]
            assert ((outs[i] - ref).norm() / ref.norm()).item() < 1e-13, runs[i]
            if s == 3:
                assert torch.equal(outs[i], eager[i])
            c, meth = runs[i]
            o = O.approx_product(M, N, sizes, c, meth, np.random.default_rng(s + i), c0=120)
            assert rel(outs[i].cpu().numpy(), o["CD"]) < 1e-12, runs[i]
    with pytest.raises(RuntimeError):
        group.pipes[0].run(Md, Nd, seeds(3)[0])


def test_pipeline_ssm_matches_oracle():
    M, N, sizes = workloads.cfg1(scale=10)
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    pipe = SketchPipeline(M.shape[0], M.shape[1], N.shape[1], sizes, 0, "SSM", draws=4)
    rng_a, rng_b = np.random.default_rng(3), np.random.default_rng(3)
    CD = pipe.run(Md, Nd, seeds_from_rngs("SSM", [rng_a], len(sizes), draws=4)).cpu().numpy()
    ref = O.ssm_product(M, N, sizes, 4, rng_b)
    assert np.array_equal(pipe.columns_host()[0], ref["blocks"])
    np.testing.assert_allclose(pipe.scales_host()[0], ref["scale"], rtol=1e-13)
    assert rel(CD, ref["CD"]) < 1e-12
    assert rng_a.bit_generator.state == rng_b.bit_generator.state


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_pipeline_batched_matches_per_problem(dtype):
    B, m, n, p, K = 5, 32, 1024, 24, 16
    Ms, Ns = [], []
    for b in range(B):
        g = np.random.default_rng(100 + b)
        Ms.append((g.standard_normal((m, n)) * g.lognormal(0, 1, n)).astype(dtype))
        Ns.append((g.standard_normal((n, p)) * g.lognormal(0, 1, (n, 1))).astype(dtype))
    Md = torch.as_tensor(np.stack(Ms), device="cuda")
    Nd = torch.as_tensor(np.stack(Ns), device="cuda")
    sizes = (n // K,) * K
    c = 256
    tol = 1e-12 if dtype == np.float64 else 1e-5  # float32 inputs run the tcgen05 3xTF32 contraction
    for method in ("ONC", "OPL"):
        pipe = SketchPipeline(m, n, p, sizes, c, method, batch=B, dtype=Md.dtype)
        assert pipe.tf32 == (dtype == np.float32)
        rngs = [workloads.sample_rng(5, b) for b in range(B)]
        CD = pipe.run(Md, Nd, seeds_from_rngs(method, rngs, K)).cpu().numpy()
        pipe.check()
        for b in range(B):
            ref = O.approx_product(Ms[b].astype(np.float64), Ns[b].astype(np.float64), sizes, c, method,
                                   workloads.sample_rng(5, b))
            assert np.array_equal(pipe.budgets_host()[b], ref["budgets"]), (method, b)
            assert np.array_equal(pipe.columns_host()[b], ref["columns"]), (method, b)
            assert np.array_equal(pipe.scales_host()[b], ref["scale"]), (method, b)
            assert rel(CD[b], ref["CD"]) < tol


def test_cfg5_subset_against_oracle():
    """Config 5 problems (float32, 256x4096 . 4096x256, K=64, W=1024): first 8 of the batch."""
    B, m, n, p, K, W = 8, 256, 4096, 256, 64, 1024
    probs = [workloads.cfg5_problem(b) for b in range(B)]
    Md = torch.as_tensor(np.stack([x[0] for x in probs]), device="cuda")
    Nd = torch.as_tensor(np.stack([x[1] for x in probs]), device="cuda")
    sizes = (64,) * K
    pipe = SketchPipeline(m, n, p, sizes, W, "ONC", batch=B, dtype=torch.float32)
    CD = pipe.run(Md, Nd, seeds_from_rngs("ONC", [workloads.sample_rng(5, b) for b in range(B)], K)).cpu().numpy()
    pipe.check()
    for b in range(B):
        M64, N64 = probs[b][0].astype(np.float64), probs[b][1].astype(np.float64)
        ref = O.approx_product(M64, N64, sizes, W, "ONC", workloads.sample_rng(5, b))
        assert np.array_equal(pipe.budgets_host()[b], ref["budgets"])
        assert np.array_equal(pipe.columns_host()[b], ref["columns"])
        assert np.array_equal(pipe.scales_host()[b], ref["scale"])
        assert rel(CD[b], ref["CD"]) < 1e-5


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("method", ["ONC", "OPL", "SSM"])
def test_sharded_world1_matches_pipeline(dtype, method):
    from paper_2105_04940_b200.distributed import ShardLayout, ShardedApproxProduct
    M, N, sizes = workloads.cfg1(scale=10)  # equal blocks (SSM)
    m, n, p = M.shape[0], M.shape[1], N.shape[1]
    Md = torch.as_tensor(M, device="cuda", dtype=dtype)
    Nd = torch.as_tensor(N, device="cuda", dtype=dtype)
    c = 8 if method == "SSM" else 512
    sh = ShardedApproxProduct(ShardLayout(1, 0, m, n, p), sizes, [(method, c)], dtype=dtype)
    out = sh.run(Md, Nd, [seeds_from_rngs(method, [np.random.default_rng(9)], len(sizes), draws=c)])[0].cpu().numpy()
    sh.check()
    pipe = (SketchPipeline(m, n, p, sizes, 0, "SSM", draws=c, dtype=dtype) if method == "SSM" else
            SketchPipeline(m, n, p, sizes, c, method, dtype=dtype))
    ref = pipe.run(Md, Nd, seeds_from_rngs(method, [np.random.default_rng(9)], len(sizes), draws=c)).cpu().numpy()
    assert np.array_equal(sh.pipes[0].columns_host(), pipe.columns_host())
    assert np.array_equal(out, ref)


def test_pipeline_reports_reference_errors():
    M, N, sizes = workloads.cfg1(scale=10)
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    pipe = SketchPipeline(M.shape[0], M.shape[1], N.shape[1], sizes, 5, "ONC")  # 5 < K floors
    pipe.run(Md, Nd, seeds_from_rngs("ONC", [np.random.default_rng(0)], len(sizes)))
    with pytest.raises(ValueError, match="required floors"):
        pipe.check()


def test_compressed_sketch_matches_draws_and_uncompressed_product():
    """bmm_compress_sketch: distinct drawn columns in column order, scale
    s_i sqrt(c_i), zero padding, count; the compressed contraction equals the
    draw-order one to rounding."""
    from paper_2105_04940_b200 import _lib
    M, N, sizes = workloads.cfg2(n=4000, m=60, p=50, K=12)
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    a = SketchPipeline(60, 4000, 50, sizes, 900, "OPL", compress=True)
    b = SketchPipeline(60, 4000, 50, sizes, 900, "OPL", compress=False)
    CDa = a.run(Md, Nd, seeds_from_rngs("OPL", [np.random.default_rng(4)], len(sizes))).cpu().numpy()
    CDb = b.run(Md, Nd, seeds_from_rngs("OPL", [np.random.default_rng(4)], len(sizes))).cpu().numpy()
    assert np.array_equal(a.columns_host(), b.columns_host())
    assert rel(CDa, CDb) < 1e-13
    cols, scales = a.columns_host()[0], a.scales_host()[0]
    uniq, counts = np.unique(cols, return_counts=True)
    kd = int(a.k_count[0].item())
    assert kd == uniq.size
    kc = a.k_column.cpu().numpy()
    ks = a.k_scale.cpu().numpy()
    pad = min(kc.size, -(-kd // 32) * 32)
    assert np.array_equal(kc[:kd], uniq) and (kc[kd:pad] == 0).all() and (ks[kd:pad] == 0).all()
    first = {c: s for c, s in zip(cols[::-1], scales[::-1])}
    assert np.allclose(ks[:kd], np.array([first[c] for c in uniq]) * np.sqrt(counts), rtol=1e-15, atol=0)
    # direct C-ABI call on a batch of 2 with a stride
    col2 = torch.as_tensor(np.stack([cols, cols[::-1].copy()]), device="cuda")
    sc2 = torch.as_tensor(np.stack([scales, scales[::-1].copy()]), device="cuda")
    W = cols.size
    oc = torch.empty(2 * W, dtype=torch.int64, device="cuda")
    os_ = torch.empty(2 * W, dtype=torch.float64, device="cuda")
    cnt = torch.empty(2, dtype=torch.int64, device="cuda")
    ws = _lib.workspace(_lib.load().bmm_compress_workspace(4000, 2))
    _lib.call("bmm_compress_sketch", col2.data_ptr(), sc2.data_ptr(), W, W, 4000, 2, ws.data_ptr(), ws.numel(),
              oc.data_ptr(), os_.data_ptr(), cnt.data_ptr(), _lib.stream_ptr())
    assert cnt.cpu().tolist() == [kd, kd]
    assert np.array_equal(oc.view(2, W)[1, :kd].cpu().numpy(), uniq)


@pytest.mark.parametrize("joint,shared", [(False, False), (True, False), (False, True), (True, True)])
def test_streamed_end_to_end_graph_matches_resident_run(joint, shared):
    """PipelineGroup.capture_host: chunked host->device transfer with the norm
    pass and OPL's segmented square sums behind it, products copied back to
    pinned host buffers -- bit-identical to the device-resident replay."""
    M, N, sizes = workloads.cfg2(n=4000, m=60, p=50, K=12)
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    runs = [(c, meth) for c in (200, 400) for meth in ("OPL", "ONC", "ONMCNR")]
    mk = lambda: PipelineGroup([SketchPipeline(60, 4000, 50, sizes, c, meth, c0=120) for c, meth in runs],  # noqa: E731
                               joint=joint, shared=shared)
    seeds = lambda s: [seeds_from_rngs(meth, [np.random.default_rng(s + i)], len(sizes))  # noqa: E731
                       for i, (c, meth) in enumerate(runs)]
    ref = mk()
    want = [o.cpu().numpy() for o in ref.run(Md, Nd, seeds(7))]
    grp = mk()
    Mh, Nh = torch.from_numpy(M).pin_memory(), torch.from_numpy(N).pin_memory()
    Mx, Nx = torch.empty_like(Md), torch.empty_like(Nd)
    outs = [torch.empty((60, 50), dtype=torch.float64).pin_memory() for _ in runs]
    grp.capture_host(Mx, Nx, Mh, Nh, outs, seeds(0), n_chunks=5)
    for rep in range(2):
        Mx.zero_()
        Nx.zero_()
        grp.run_host(seeds(7))
        torch.cuda.synchronize()
        for o, w in zip(outs, want):
            assert np.array_equal(o.numpy(), w)
    assert np.array_equal(Mx.cpu().numpy(), M)


@pytest.mark.parametrize("serial", ["0", "1"])
def test_streamed_end_to_end_float32_shared_group(serial, monkeypatch):
    """The config-4 end-to-end shape at small size: float32 host inputs streamed in
    chunks under the shared statistics stage (norms and Gram g_k per chunk), OPL,
    ONC and SSM members, products copied back -- bit-identical to the resident run."""
    g = np.random.default_rng(8)
    sizes = (64,) * 48
    n = sum(sizes)
    M = (g.standard_normal((72, n)) * np.repeat(g.uniform(0.1, 10, 48), 64)).astype(np.float32)
    N = (g.standard_normal((n, 40)) * np.repeat(g.uniform(0.1, 10, 48), 64)[:, None]).astype(np.float32)
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    mk = lambda: PipelineGroup([SketchPipeline(72, n, 40, sizes, 768, "OPL", dtype=torch.float32),  # noqa: E731
                                SketchPipeline(72, n, 40, sizes, 768, "ONC", dtype=torch.float32),
                                SketchPipeline(72, n, 40, sizes, 0, "SSM", draws=12, dtype=torch.float32)])

    def seeds(s):
        return [seeds_from_rngs("OPL", [np.random.default_rng(s)], 48),
                seeds_from_rngs("ONC", [np.random.default_rng(s + 1)], 48),
                seeds_from_rngs("SSM", [np.random.default_rng(s + 2)], 48, draws=12)]

    monkeypatch.setenv("BMM_GROUP_SERIAL", serial)
    want = [o.cpu().numpy() for o in mk().run(Md, Nd, seeds(4))]
    grp = mk()
    Mh, Nh = torch.from_numpy(M).pin_memory(), torch.from_numpy(N).pin_memory()
    Mx, Nx = torch.empty_like(Md), torch.empty_like(Nd)
    outs = [torch.empty((72, 40), dtype=torch.float32).pin_memory() for _ in range(3)]
    grp.capture_host(Mx, Nx, Mh, Nh, outs, seeds(0), n_chunks=6)
    for _ in range(2):
        Mx.zero_()
        Nx.zero_()
        grp.run_host(seeds(4))
        torch.cuda.synchronize()
        for o, w in zip(outs, want):
            assert np.array_equal(o.numpy(), w)


@pytest.mark.parametrize("bad", [np.nan, np.inf])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_nonfinite_input_raises_like_the_reference(bad, dtype):
    """NaN/Inf in M: the pipeline reports the reference's exception (first bad
    block's probabilities for OPL/ONC, integerize's weights for the two-step
    plan, empty support for SSM) and never indexes outside the inputs."""
    M, N, sizes = workloads.cfg1(scale=10)  # 200 x 1000, ten equal blocks of 100 (SSM needs equal blocks)
    M = M.astype(dtype)
    N = N.astype(dtype)
    M[7, 2 * 100 + 5] = bad  # a column of block 2
    m, n, p = M.shape[0], M.shape[1], N.shape[1]
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    want = {"OPL": "block 2: probabilities must be finite", "ONC": "block 2: probabilities must be finite",
            "ONU": "weights must be finite", "SSM": "probability vector has empty support"}
    for meth, msg in want.items():
        pipe = (SketchPipeline(m, n, p, sizes, 0, "SSM", draws=5, dtype=tdt) if meth == "SSM" else
                SketchPipeline(m, n, p, sizes, 400, meth, c0=40, dtype=tdt))
        pipe.run(Md, Nd, seeds_from_rngs(meth, [np.random.default_rng(1)], len(sizes), draws=5))
        torch.cuda.synchronize()
        with pytest.raises(ValueError, match=msg):
            pipe.check()
    torch.cuda.synchronize()


@pytest.mark.parametrize("method", ["ONC", "OPL", "SSM"])
def test_many_small_blocks_thread_kernels_match_oracle(method):
    """K x batch >= 16384 blocks of <= 64 columns take the thread-per-block
    probability and sampling kernels (config 5's shape): budgets, draws and
    scales bit-exact to the oracle on a spread of problems, with a zero block."""
    B, m, n, p, K = 260, 24, 4096, 16, 64
    g = np.random.default_rng(31)
    Ms = (g.standard_normal((B, m, n)) * g.lognormal(0, 1, (B, 1, n))).astype(np.float32)
    Ns = (g.standard_normal((B, n, p)) * g.lognormal(0, 1, (B, n, 1))).astype(np.float32)
    sizes = (64,) * K
    if method != "SSM":
        Ms[:, :, 64:128] = 0.0  # block 1 has zero score in every problem
    Md, Nd = torch.as_tensor(Ms, device="cuda"), torch.as_tensor(Ns, device="cuda")
    if method == "SSM":
        pipe = SketchPipeline(m, n, p, sizes, 0, "SSM", batch=B, draws=8, dtype=torch.float32)
        rngs = [np.random.default_rng(1000 + b) for b in range(B)]
        CD = pipe.run(Md, Nd, seeds_from_rngs("SSM", rngs, K, draws=8)).cpu().numpy()
    else:
        pipe = SketchPipeline(m, n, p, sizes, 512, method, batch=B, dtype=torch.float32)
        rngs = [np.random.default_rng(1000 + b) for b in range(B)]
        CD = pipe.run(Md, Nd, seeds_from_rngs(method, rngs, K)).cpu().numpy()
    pipe.check()
    for b in (0, 1, 77, 130, 259):
        M64, N64 = Ms[b].astype(np.float64), Ns[b].astype(np.float64)
        if method == "SSM":
            ref = O.ssm_product(M64, N64, sizes, 8, np.random.default_rng(1000 + b))
            assert np.array_equal(pipe.columns_host()[b], ref["blocks"]), b
        else:
            ref = O.approx_product(M64, N64, sizes, 512, method, np.random.default_rng(1000 + b))
            assert np.array_equal(pipe.budgets_host()[b], ref["budgets"]), b
            assert np.array_equal(pipe.columns_host()[b], ref["columns"]), b
            assert np.array_equal(pipe.scales_host()[b], ref["scale"]), b
        assert rel(CD[b], ref["CD"]) < 1e-5


@pytest.mark.parametrize("method", ["ONC", "OPL", "SSM"])
def test_waves_bit_identical_to_single_batch(method):
    """set_waves: the batch as sub-batches on several streams (uneven last wave),
    eager and as one captured graph -- products, budgets, draws and scales are
    bit-identical to the single-batch launch; seeds changed between replays."""
    B, m, n, p, K = 23, 256, 1024, 256, 16
    g = np.random.default_rng(77)
    Ms = (g.standard_normal((B, m, n)) * g.lognormal(0, 1, (B, 1, n))).astype(np.float32)
    Ns = (g.standard_normal((B, n, p)) * g.lognormal(0, 1, (B, n, 1))).astype(np.float32)
    sizes = (64,) * K
    Md, Nd = torch.as_tensor(Ms, device="cuda"), torch.as_tensor(Ns, device="cuda")

    def make():
        if method == "SSM":
            return SketchPipeline(m, n, p, sizes, 0, "SSM", batch=B, draws=4, dtype=torch.float32)
        return SketchPipeline(m, n, p, sizes, 256, method, batch=B, dtype=torch.float32)

    def seeds(base):
        rngs = [np.random.default_rng(base + b) for b in range(B)]
        return seeds_from_rngs(method, rngs, K, draws=4) if method == "SSM" else seeds_from_rngs(method, rngs, K)

    ref, wav = make(), make()
    assert wav.fused16
    wav.set_waves(5, 3)
    for rnd, base in enumerate((500, 900, 1300)):
        if rnd == 1:
            wav.capture(Md, Nd)  # later rounds replay the multi-stream graph
        CDr = ref.run(Md, Nd, seeds(base)).clone()
        CDw = wav.run(Md, Nd, seeds(base)).clone()
        ref.check()
        wav.check()
        assert torch.equal(CDr, CDw), (method, rnd)
        assert np.array_equal(ref.columns_host(), wav.columns_host())
        assert np.array_equal(ref.scales_host(), wav.scales_host())
        if method != "SSM":
            assert np.array_equal(ref.budgets_host(), wav.budgets_host())
    with pytest.raises(ValueError, match="waves"):
        SketchPipeline(40, 512, 40, (64,) * 8, 128, "ONC", batch=4).set_waves(2, 2)


@pytest.mark.parametrize("method,dtype", [("ONC", "f32"), ("OPL", "f32"), ("ONC", "f64"), ("OPL", "f64")])
def test_plan_small_matches_separate_kernels(method, dtype, monkeypatch):
    """bmm_plan_small (probabilities, budgets, child streams, draws, compressed sketch and
    balanced exponents of a problem in one CTA) against the separate kernels: every plan
    output bit-identical, unequal blocks, a zero-score block, an all-zero problem (its
    status raises the reference's error), and the oracle on a few problems."""
    B, m, n, p = 300, 24, 1000, 16
    sizes = (64, 1, 100, 35, 128, 64, 8, 90, 64, 64, 64, 31, 97, 64, 62, 64)
    assert sum(sizes) == n
    K = len(sizes)
    g = np.random.default_rng(5)
    npdt = np.float32 if dtype == "f32" else np.float64
    Ms = (g.standard_normal((B, m, n)) * g.lognormal(0, 1, (B, 1, n))).astype(npdt)
    Ns = (g.standard_normal((B, n, p)) * g.lognormal(0, 1, (B, n, 1))).astype(npdt)
    Ms[:, :, 65:165] = 0.0  # block 2 has zero score in every problem
    Ms[7] = 0.0             # problem 7: nothing to sample
    Md, Nd = torch.as_tensor(Ms, device="cuda"), torch.as_tensor(Ns, device="cuda")
    tdt = torch.float32 if dtype == "f32" else torch.float64
    W = 256
    fused = SketchPipeline(m, n, p, sizes, W, method, batch=B, dtype=tdt)
    assert fused.plan_small
    waved = None
    if dtype == "f32" and fused.fused and method == "ONC":  # the two-stream pipeline over waves (norms | plan | contraction)
        waved = SketchPipeline(m, n, p, sizes, W, method, batch=B, dtype=tdt)
        waved.set_waves(128, 2)
    monkeypatch.setenv("BMM_PLAN_SMALL", "0")
    sep = SketchPipeline(m, n, p, sizes, W, method, batch=B, dtype=tdt)
    assert not sep.plan_small
    for base in (1000, 5000):
        rngs = lambda: [np.random.default_rng(base + b) for b in range(B)]  # noqa: E731
        CDf = fused.run(Md, Nd, seeds_from_rngs(method, rngs(), K)).clone()
        CDs = sep.run(Md, Nd, seeds_from_rngs(method, rngs(), K)).clone()
        for name in ("s", "probs", "last", "budgets", "col_off", "status", "diag", "notes", "states"):
            a, b_ = getattr(fused, name), getattr(sep, name)
            assert torch.equal(a, b_), (name, base)
        st = fused.status.cpu().numpy()
        assert st[7] != 0 and (np.delete(st, 7) == 0).all()
        kc = fused.k_count.cpu().numpy()
        ok = np.flatnonzero(st == 0)
        assert np.array_equal(kc[ok], sep.k_count.cpu().numpy()[ok]) and kc[7] == 0
        for name in ("column", "prob", "scale"):  # a failed plan draws nothing: its rows are not written
            a, b_ = getattr(fused, name).view(B, W), getattr(sep, name).view(B, W)
            assert torch.equal(a[ok], b_[ok]), (name, base)
        for b in ok[:40]:
            pad = min(W, (kc[b] + 63) // 64 * 64)
            sl = slice(b * W, b * W + pad)
            assert torch.equal(fused.k_column[sl], sep.k_column[sl]) and torch.equal(fused.k_scale[sl], sep.k_scale[sl])
            if hasattr(fused, "gshift"):
                assert torch.equal(fused.kexp[b * W:b * W + kc[b]], sep.kexp[b * W:b * W + kc[b]])
        if hasattr(fused, "gshift"):
            assert torch.equal(fused.gshift[ok], sep.gshift[ok])
        okt = torch.as_tensor(ok, device="cuda")
        assert torch.equal(CDf.view(B, m, p)[okt], CDs.view(B, m, p)[okt])
        if waved is not None:
            if base == 5000:
                waved.capture(Md, Nd)
            CDw = waved.run(Md, Nd, seeds_from_rngs(method, rngs(), K)).clone()
            assert torch.equal(CDw.view(B, m, p)[okt], CDf.view(B, m, p)[okt])
            assert torch.equal(waved.column.view(B, W)[okt], fused.column.view(B, W)[okt])
            assert torch.equal(waved.budgets, fused.budgets) and torch.equal(waved.status, fused.status)
    with pytest.raises(ValueError):
        fused.check()
    for b in (0, 150, 299):
        ref = O.approx_product(Ms[b].astype(np.float64), Ns[b].astype(np.float64), sizes, W, method,
                               np.random.default_rng(5000 + b))
        assert np.array_equal(fused.budgets_host()[b], ref["budgets"]), b
        assert np.array_equal(fused.columns_host()[b], ref["columns"]), b
        assert np.array_equal(fused.scales_host()[b], ref["scale"]), b
