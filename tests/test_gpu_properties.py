"""Algorithm-level properties of the device path, in the spirit of the
reference's own property tests (budget conservation, scale equivariance,
unbiasedness, large-pilot two-step ~ optimal sizes, exactness for one-column
blocks), plus a cross-check of the two widened rows against each other: the
Monte Carlo mean squared error of the replication engine (§8 f1) must match
the closed-form expected squared error (§8 f2)."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
bm = pytest.importorskip("paper_2105_04940_b200")
from paper_2105_04940_b200 import montecarlo as mc  # noqa: E402
from paper_2105_04940_b200 import variance as va  # noqa: E402


def _instance(m=30, n=400, p=20, K=8):
    return workloads.cfg2(n=n, m=m, p=p, K=K)


def test_budget_conservation_across_allocators():
    M, N, sizes = _instance()
    part = bm.BlockPartition(sizes)
    for c in (len(sizes), 57, 200, sum(sizes)):
        for plan in (bm.allocate_optimal(M, N, part, c), bm.allocate_by_score_sums(M, N, part, c),
                     bm.allocate_uniform(part, c)):
            assert plan.total == c and (plan.budgets <= np.asarray(sizes)).all() and (plan.budgets >= 1).all()
        two = bm.estimate_product_two_step(M, N, part, c, 4 * len(sizes), np.random.default_rng(c), pilot="norm")
        assert two.plan.total == c


def test_scale_equivariance_exact_for_powers_of_two():
    M, N, sizes = _instance(m=25, p=17)
    part = bm.BlockPartition(sizes)
    plan = bm.allocate_optimal(M, N, part, 120)
    plan8 = bm.allocate_optimal(8.0 * M, 0.25 * N, part, 120)
    assert np.array_equal(plan.budgets, plan8.budgets)
    for a, b in zip(plan.probs.per_block, plan8.probs.per_block):
        assert np.array_equal(a, b)
    _, cd, log = bm.estimate_product(M, N, plan, np.random.default_rng(3))
    _, cd8, log8 = bm.estimate_product(8.0 * M, 0.25 * N, plan8, np.random.default_rng(3))
    assert np.array_equal(log.column, log8.column)
    assert np.array_equal(cd8, 2.0 * cd)


def test_one_column_blocks_are_exact():
    g = np.random.default_rng(5)
    M, N = g.standard_normal((9, 6)), g.standard_normal((6, 4))
    part = bm.BlockPartition((1,) * 6)
    plan = bm.allocate_by_score_sums(M, N, part, 6)
    _, cd, _ = bm.estimate_product(M, N, plan, np.random.default_rng(0))
    assert np.allclose(cd, M @ N, rtol=1e-13, atol=1e-13)


def test_large_pilot_two_step_tracks_optimal_sizes():
    M, N, sizes = _instance(m=40, n=600, p=30, K=6)
    part = bm.BlockPartition(sizes)
    opt = bm.allocate_optimal(M, N, part, 240).budgets
    two = bm.estimate_product_two_step(M, N, part, 240, 600 * 40, np.random.default_rng(1), pilot="norm").plan.budgets
    assert np.abs(two - opt).max() <= max(2, int(0.05 * opt.max()))


@pytest.mark.parametrize("meth", ["OPL", "ONC", "UU"])
def test_monte_carlo_mse_matches_closed_form_and_mean_is_unbiased(meth):
    M, N, sizes = _instance(m=24, n=300, p=16, K=6)
    part = bm.BlockPartition(sizes)
    c = 60
    plan = {"OPL": bm.allocate_optimal, "ONC": bm.allocate_by_score_sums}.get(
        meth, lambda M_, N_, p_, c_: bm.allocate_uniform(p_, c_))(M, N, part, c)
    reps = 20000
    out = mc.ReplicationEngine(M, N, plan).run(np.random.default_rng(9), reps)
    sq = out["sq_error"].cpu().numpy()
    ese = va.expected_sq_error(M, N, plan)
    # mean of reps i.i.d. squared errors: within 5 standard errors of the closed form
    assert abs(sq.mean() - ese) < 5 * sq.std(ddof=1) / np.sqrt(reps)
    # elementwise variance sums to the expected squared error
    assert np.isclose(va.elementwise_variance(M, N, plan).sum(), ese, rtol=1e-10)
