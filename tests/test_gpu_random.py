"""Randomised parity sweep: random shapes, partitions (size-1 blocks, very
unequal blocks), zero columns / rows / blocks, float64 and float32, every
method, through both the per-call API and the device pipeline -- against the
NumPy oracle (bit-exact indices, budgets, probabilities, scales; C.D within
1e-12 float64 / 1e-5 float32)."""
import numpy as np
import pytest

from oracle import blockmm_oracle as O
from random_cases import sweep_params

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
bm = pytest.importorskip("paper_2105_04940_b200")
from paper_2105_04940_b200.pipeline import SketchPipeline, seeds_from_rngs  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    r = np.linalg.norm(b)
    return np.linalg.norm(a - b) / r if r else np.linalg.norm(a - b)


@pytest.mark.parametrize("seed", range(40))
def test_random_api_parity(seed):
    M, N, sizes, c, c0 = sweep_params(seed)
    part = bm.BlockPartition(sizes)
    cs, rs, probs, s = O.instance_stats(M, N, sizes)
    assert np.array_equal(np.concatenate(bm.optimal_probabilities(M, N, part).per_block), probs)
    assert np.array_equal(bm.score_sums(M, N, part), s)
    if not (s > 0).any():
        with pytest.raises(ValueError):
            bm.allocate_by_score_sums(M, N, part, 5)
        return
    for meth, fn in (("ONC", bm.allocate_by_score_sums), ("OPL", bm.allocate_optimal),
                     ("UU", lambda M_, N_, p_, c_: bm.allocate_uniform(p_, c_))):
        want = outcome(lambda: O.approx_product(M, N, sizes, c, meth, np.random.default_rng(seed)))
        if isinstance(want, type):
            with pytest.raises(want):
                fn(M, N, part, c)
            continue
        plan = fn(M, N, part, c)
        assert np.array_equal(plan.budgets, want["budgets"]), (seed, meth)
        _, prod, log = bm.estimate_product(M, N, plan, np.random.default_rng(seed))
        assert np.array_equal(log.column, want["columns"]), (seed, meth)
        assert np.array_equal(log.scale, want["scale"]), (seed, meth)
        assert rel(prod, want["CD"]) < 1e-12
    for meth, pil in (("ONU", "uniform"), ("ONMCNR", "norm")):
        two_step_case(M, N, sizes, part, c, c0, seed, meth, pil)


def outcome(fn):
    """fn()'s value, or the reference exception class it raised (ValueError /
    AssertionError; the oracle's OracleAssert is reported as AssertionError)."""
    try:
        return fn()
    except AssertionError:
        return AssertionError
    except ValueError:
        return ValueError


def two_step_case(M, N, sizes, part, c, c0, seed, meth, pil):
    """Two-step parity.  The pilot draws are bit-exact and the pilot norms agree
    to rounding (BLAS order in the reference).  The budgets are a discontinuous
    function of sqrt|s^2 - pilot^2|, which is pure rounding noise when a pilot
    sketch reproduces s_k exactly in real arithmetic (one pilot draw per block:
    ||M_i N_i^T||_F / p_i == s_k), in the reference itself.  So: budgets (or
    the raised error) must equal the oracle's integerisation of OUR pilot norms
    bit for bit, and equal the oracle end to end whenever its own pilot norms
    give the same plan."""
    K = len(sizes)
    ref_psq = O.two_step_pilot(M, N, sizes, c0, meth, np.random.default_rng(seed))[0]
    pipe = SketchPipeline(M.shape[0], M.shape[1], N.shape[1], sizes, c, meth, batch=1,
                          dtype=torch.float64, c0=c0)
    pipe.run(torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda"),
             seeds_from_rngs(meth, [np.random.default_rng(seed)], K))
    our_psq = pipe.pilot_sq.cpu().numpy()
    assert np.allclose(our_psq, ref_psq, rtol=1e-12, atol=0.0), (seed, meth, our_psq, ref_psq)
    s = O.instance_stats(M, N, sizes)[3]
    want = outcome(lambda: O.plan_budgets("TWO_STEP", sizes, c, s=s, aux_sq=our_psq)[0])
    got = outcome(lambda: bm.estimate_product_two_step(M, N, part, c, c0, np.random.default_rng(seed),
                                                       pilot=pil))
    if isinstance(want, type):
        assert got is want, (seed, meth, got)
        return
    assert not isinstance(got, type), (seed, meth, got)
    assert np.array_equal(got.plan.budgets, want), (seed, meth)
    assert np.array_equal(got.plan.pilot_norms ** 2, our_psq) or np.allclose(
        got.plan.pilot_norms ** 2, our_psq, rtol=1e-15, atol=0.0)
    ref = outcome(lambda: O.approx_product(M, N, sizes, c, meth, np.random.default_rng(seed), c0=c0))
    if isinstance(ref, type) or not np.array_equal(ref["budgets"], want):
        return  # ill-conditioned pilot weights: plan differs by rounding only
    assert np.array_equal(got.log.column, ref["columns"]), (seed, meth)
    assert rel(got.product, ref["CD"]) < 1e-12


@pytest.mark.parametrize("seed", range(16))
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
    if seed >= 8:  # widths off the 8-column pair groups: float32 takes the float64 gather + DMMA path
        c = int(min(n, max(K, c - 3)))
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
