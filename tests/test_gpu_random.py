"""Randomised parity sweep: random shapes, partitions (size-1 blocks, very
unequal blocks), zero columns / rows / blocks, float64 and float32, every
method, through both the per-call API and the device pipeline -- against the
NumPy oracle (bit-exact indices, budgets, probabilities, scales; C.D within
1e-12 float64 / 1e-5 float32)."""
import numpy as np
import pytest

from oracle import blockmm_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
bm = pytest.importorskip("paper_2105_04940_b200")
from paper_2105_04940_b200.pipeline import SketchPipeline, seeds_from_rngs  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    r = np.linalg.norm(b)
    return np.linalg.norm(a - b) / r if r else np.linalg.norm(a - b)


def random_instance(g):
    K = int(g.integers(1, 24))
    kind = g.integers(0, 3)
    if kind == 0:
        sizes = g.integers(1, 40, K)
    elif kind == 1:
        sizes = np.maximum(1, (g.lognormal(3, 1.2, K)).astype(int))
    else:
        sizes = np.full(K, int(g.integers(1, 64)))
    n = int(sizes.sum())
    m, p = int(g.integers(1, 70)), int(g.integers(1, 70))
    M = g.standard_normal((m, n)) * g.lognormal(0, 1.5, n)
    N = g.standard_normal((n, p)) * g.lognormal(0, 1.5, (n, 1))
    if g.random() < 0.3:
        M[:, g.integers(0, n, max(1, n // 10))] = 0.0
    if g.random() < 0.2 and K > 1:
        k = int(g.integers(0, K))
        o = int(sizes[:k].sum())
        N[o:o + sizes[k]] = 0.0
    return M, N, tuple(int(s) for s in sizes)


@pytest.mark.parametrize("seed", range(12))
def test_random_api_parity(seed):
    g = np.random.default_rng(1000 + seed)
    M, N, sizes = random_instance(g)
    K = len(sizes)
    part = bm.BlockPartition(sizes)
    cs, rs, probs, s = O.instance_stats(M, N, sizes)
    assert np.array_equal(np.concatenate(bm.optimal_probabilities(M, N, part).per_block), probs)
    assert np.array_equal(bm.score_sums(M, N, part), s)
    live = int((s > 0).sum())
    if live == 0:
        with pytest.raises(ValueError):
            bm.allocate_by_score_sums(M, N, part, 5)
        return
    caps = np.where(s > 0, np.asarray(sizes), 0)
    c = int(g.integers(live, max(live, int(caps.sum())) + 1))
    for meth, fn in (("ONC", bm.allocate_by_score_sums), ("OPL", bm.allocate_optimal)):
        try:
            ref = O.approx_product(M, N, sizes, c, meth, np.random.default_rng(seed))
        except (ValueError, AssertionError) as exc:
            with pytest.raises(type(exc)):
                fn(M, N, part, c)
            continue
        plan = fn(M, N, part, c)
        assert np.array_equal(plan.budgets, ref["budgets"]), (seed, meth)
        _, prod, log = bm.estimate_product(M, N, plan, np.random.default_rng(seed))
        assert np.array_equal(log.column, ref["columns"]), (seed, meth)
        assert np.array_equal(log.scale, ref["scale"]), (seed, meth)
        assert rel(prod, ref["CD"]) < 1e-12
    c0 = K * int(g.integers(1, 4))
    for meth, pil in (("ONU", "uniform"), ("ONMCNR", "norm")):
        try:
            ref = O.approx_product(M, N, sizes, c, meth, np.random.default_rng(seed), c0=c0)
        except (ValueError, AssertionError) as exc:
            with pytest.raises(type(exc)):
                bm.estimate_product_two_step(M, N, part, c, c0, np.random.default_rng(seed), pilot=pil)
            continue
        res = bm.estimate_product_two_step(M, N, part, c, c0, np.random.default_rng(seed), pilot=pil)
        assert np.array_equal(res.plan.budgets, ref["budgets"]), (seed, meth)
        assert np.array_equal(res.log.column, ref["columns"]), (seed, meth)
        assert rel(res.product, ref["CD"]) < 1e-12


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_random_pipeline_parity(seed, dtype):
    g = np.random.default_rng(2000 + seed)
    B = int(g.integers(1, 5))
    K = int(g.integers(1, 20))
    sizes = tuple(int(x) for x in g.integers(1, 50, K))
    n = sum(sizes)
    m, p = int(g.integers(8, 200)), int(g.integers(8, 200))
    Ms = [(g.standard_normal((m, n)) * g.lognormal(0, 1, n)).astype(dtype) for _ in range(B)]
    Ns = [(g.standard_normal((n, p)) * g.lognormal(0, 1, (n, 1))).astype(dtype) for _ in range(B)]
    c = 8 * int(g.integers(max(1, (K + 7) // 8), max(2, n // 8) + 1))
    method = ["ONC", "OPL", "UU", "ONU", "ONMCNR"][seed % 5]
    c0 = 2 * K
    Md = torch.as_tensor(np.stack(Ms), device="cuda")
    Nd = torch.as_tensor(np.stack(Ns), device="cuda")
    pipe = SketchPipeline(m, n, p, sizes, c, method, batch=B, dtype=Md.dtype, c0=c0)
    rngs = [np.random.default_rng(seed * 10 + b) for b in range(B)]
    CD = pipe.run(Md, Nd, seeds_from_rngs(method, rngs, K)).cpu().numpy().reshape(B, m, p)
    for b in range(B):
        M64, N64 = Ms[b].astype(np.float64), Ns[b].astype(np.float64)
        try:
            ref = O.approx_product(M64, N64, sizes, c, method, np.random.default_rng(seed * 10 + b), c0=c0)
        except (ValueError, AssertionError):
            with pytest.raises((ValueError, AssertionError)):
                pipe.check()
            return
        assert np.array_equal(pipe.budgets_host()[b], ref["budgets"]), (seed, b, method)
        assert np.array_equal(pipe.columns_host()[b], ref["columns"]), (seed, b, method)
        assert rel(CD[b], ref["CD"]) < (1e-12 if dtype == np.float64 else 1e-5)
    pipe.check()
