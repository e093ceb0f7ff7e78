"""Device Monte Carlo replication engine and exact variance analytics
 against the reference's golden outputs
(tests/golden/analytics.npz): replication draws bit-exact, squared errors,
variances and expectations to rounding, coverage counts identical."""
from pathlib import Path

import numpy as np
import pytest

from random_cases import sweep_params

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
bm = pytest.importorskip("paper_2105_04940_b200")
from paper_2105_04940_b200 import montecarlo as mc  # noqa: E402
from paper_2105_04940_b200 import variance as va  # noqa: E402

G = np.load(Path(__file__).resolve().parent / "golden" / "analytics.npz")
SEEDS = sorted({int(k.split("_")[0][1:]) for k in G.files if k.startswith("s") and "__" in k})


def _plan(M, N, part, c, meth):
    if meth == "UU":
        return bm.allocate_uniform(part, c)
    return (bm.allocate_optimal if meth == "OPL" else bm.allocate_by_score_sums)(M, N, part, c)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("meth", ["ONC", "OPL", "UU"])
def test_variance_and_replications_match_reference(seed, meth):
    M, N, sizes, c, _ = sweep_params(seed)
    part = bm.BlockPartition(sizes)
    key = f"s{seed}_{meth}"
    plan = _plan(M, N, part, c, meth)
    assert np.array_equal(plan.budgets, G[key + "__budgets"])
    assert rel(va.elementwise_variance(M, N, plan), G[key + "__var"]) < 1e-10
    assert np.isclose(va.expected_sq_error(M, N, plan), G[key + "__ese"][0], rtol=1e-10)
    reps = len(G[key + "__rep_sq"])
    rng = np.random.default_rng(100 + seed)
    out = mc.ReplicationEngine(M, N, plan, chunk=37).run(rng, reps, keep_columns=True)
    assert rng.bit_generator.seed_seq.n_children_spawned == reps  # rng.spawn(reps) side effect
    assert np.array_equal(out["columns"].cpu().numpy(), G[key + "__rep_cols"])
    assert np.allclose(out["sq_error"].cpu().numpy(), G[key + "__rep_sq"], rtol=1e-10, atol=0)
    bound, viol, lo, hi = G[key + "__coverage"]
    cov = mc.coverage_check_plan(M, N, plan, bound, reps, np.random.default_rng(100 + seed))
    assert cov.violations == int(viol) and np.isclose(cov.ci_low, lo) and np.isclose(cov.ci_high, hi)


@pytest.mark.parametrize("seed", SEEDS)
def test_minimum_expected_sq_error(seed):
    M, N, sizes, c, _ = sweep_params(seed)
    assert np.isclose(va.minimum_expected_sq_error(M, N, bm.BlockPartition(sizes), c), G[f"s{seed}__mese"][0],
                      rtol=1e-10)


def test_normality_diagnostic_matches_reference():
    M, N, sizes, c, _ = sweep_params(7)
    plan = bm.allocate_optimal(M, N, bm.BlockPartition(sizes), c)
    res = mc.normality_diagnostic(M, N, plan, (1, 2), len(G["normal__samples"]), np.random.default_rng(9))
    assert np.allclose(res.samples, G["normal__samples"], rtol=0, atol=1e-8)
    assert np.allclose([res.mean, res.variance, res.ks_distance], G["normal__stats"], rtol=1e-6, atol=1e-9)


def test_generic_runner_coverage_equals_plan_engine():
    M, N, sizes, c, _ = sweep_params(4)
    plan = bm.allocate_by_score_sums(M, N, bm.BlockPartition(sizes), c)
    bound = float(G["s4_ONC__coverage"][0])
    a = mc.coverage_check(M, N, 120, np.random.default_rng(104),
                          lambda s: (bm.estimate_product(M, N, plan, s)[1], bound))
    b = mc.coverage_check_plan(M, N, plan, bound, 120, np.random.default_rng(104))
    assert a == b


def test_analytics_errors_like_reference():
    M, N, sizes, c, _ = sweep_params(4)
    part = bm.BlockPartition(sizes)
    plan = bm.allocate_by_score_sums(M, N, part, c)
    with pytest.raises(ValueError, match="at least 100"):
        mc.coverage_check_plan(M, N, plan, 1.0, 99, np.random.default_rng(0))
    with pytest.raises(ValueError, match="budget override"):
        va.elementwise_variance(M, N, plan, budgets=np.ones(part.num_blocks + 1))
    zero = np.array(plan.budgets, dtype=float)
    zero[0] = 0.0  # block 0 has sampling variance
    with pytest.raises(ValueError, match="block 0: zero budget on a block with sampling variance"):
        va.expected_sq_error(M, N, plan, budgets=zero)
    with pytest.raises(ValueError, match="block 0: zero budget on a block with sampling variance"):
        va.elementwise_variance(M, N, plan, budgets=zero)
    with pytest.raises(ValueError, match="budget must be positive"):
        va.minimum_expected_sq_error(M, N, part, 0)
