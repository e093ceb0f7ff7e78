"""Pin the oracle's Monte Carlo replication and exact-variance restatements
 against the reference's own outputs
(tests/golden/analytics.npz, made by tests/golden/make_analytics.py).  CPU only."""
from pathlib import Path

import numpy as np
import pytest

from oracle import blockmm_oracle as O
from random_cases import sweep_params

G = np.load(Path(__file__).resolve().parent / "golden" / "analytics.npz")
SEEDS = sorted({int(k.split("_")[0][1:]) for k in G.files if k.startswith("s") and "__" in k})


def _plan(M, N, sizes, c, meth):
    _, _, probs, s = O.instance_stats(M, N, sizes)
    if meth == "UU":
        probs = np.concatenate([np.full(nk, 1.0 / nk) for nk in sizes])
        return probs, O.plan_budgets("UU", sizes, c)[0]
    aux = O.block_product_sq(M, N, sizes) if meth == "OPL" else None
    return probs, O.plan_budgets(meth, sizes, c, s=s, aux_sq=aux)[0]


@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("meth", ["ONC", "OPL", "UU"])
def test_oracle_analytics_match_reference(seed, meth):
    M, N, sizes, c, _ = sweep_params(seed)
    key = f"s{seed}_{meth}"
    probs, budgets = _plan(M, N, sizes, c, meth)
    assert np.array_equal(budgets, G[key + "__budgets"])
    var = O.elementwise_variance(M, N, sizes, probs, budgets)
    ref = G[key + "__var"]
    assert np.linalg.norm(var - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.isclose(O.expected_sq_error(M, N, sizes, probs, budgets), G[key + "__ese"][0], rtol=1e-12)
    rep = O.replicate(M, N, sizes, probs, budgets, np.random.default_rng(100 + seed), len(G[key + "__rep_sq"]))
    assert np.array_equal(rep["columns"], G[key + "__rep_cols"])
    assert np.allclose(rep["sq_error"], G[key + "__rep_sq"], rtol=1e-12, atol=0)
    bound, viol = G[key + "__coverage"][:2]
    assert int((rep["sq_error"] > bound).sum()) == int(viol)


def test_oracle_normality_replications_match_reference():
    M, N, sizes, c, _ = sweep_params(7)
    probs, budgets = _plan(M, N, sizes, c, "OPL")
    reps = len(G["normal__samples"])
    rep = O.replicate(M, N, sizes, probs, budgets, np.random.default_rng(9), reps, entry=(1, 2))
    sigma = np.sqrt(O.elementwise_variance(M, N, sizes, probs, budgets)[1, 2])
    samples = (rep["entry"] - (M @ N)[1, 2]) / sigma
    assert np.allclose(samples, G["normal__samples"], rtol=0, atol=1e-9)
