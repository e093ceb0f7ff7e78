"""Golden outputs of the reference's Monte Carlo and exact-variance functions
(pkg/src/blockmm/analysis.py:57-125, 343-416) on small
seeded instances from tests/random_cases.py.

Runs the REFERENCE package (``blockmm`` from /root/reference/pkg/src), so it
only works in the build container; the .npz output is committed.  Re-run with

    python tests/golden/make_analytics.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import blockmm as ref  # noqa: E402  (the reference, read-only)
from blockmm import analysis as ra  # noqa: E402

from random_cases import sweep_params  # noqa: E402

SEEDS = (2, 4, 5, 11)
REPS = 120
NORMAL_SEED, NORMAL_REPS = 7, 1000


def plans(M, N, part, c):
    return {"ONC": ref.allocate_by_score_sums(M, N, part, c), "OPL": ref.allocate_optimal(M, N, part, c),
            "UU": ref.allocate_uniform(part, c)}


def main():
    out = {}
    for seed in SEEDS:
        M, N, sizes, c, _ = sweep_params(seed)
        part = ref.BlockPartition(sizes)
        for meth, plan in plans(M, N, part, c).items():
            key = f"s{seed}_{meth}"
            out[key + "__budgets"] = plan.budgets
            out[key + "__var"] = ra.elementwise_variance(M, N, plan)
            out[key + "__ese"] = np.array([ra.expected_sq_error(M, N, plan)])
            # replications exactly as coverage_check runs them (analysis.py:359-362)
            rng = np.random.default_rng(100 + seed)
            exact = ref.multiply_exact(M, N)
            sq, cols = [], []
            for stream in rng.spawn(REPS):
                _, est, log = ref.estimate_product(M, N, plan, stream)
                sq.append(ref.frobenius_norm(est - exact) ** 2)
                cols.append(log.column)
            out[key + "__rep_sq"] = np.array(sq)
            out[key + "__rep_cols"] = np.array(cols)
            bound = float(np.quantile(sq, 0.8))
            cov = ra.coverage_check_plan(M, N, plan, bound, REPS, np.random.default_rng(100 + seed))
            out[key + "__coverage"] = np.array([bound, cov.violations, cov.ci_low, cov.ci_high])
        out[f"s{seed}__mese"] = np.array([ra.minimum_expected_sq_error(M, N, part, c)])
        # closed-form bounds (analysis.py:148-315), incl. a two-step plan's pilot bound
        two = ref.estimate_product_two_step(M, N, part, c, 3 * len(sizes), np.random.default_rng(seed),
                                            pilot="uniform").plan
        for meth, plan in list(plans(M, N, part, c).items()) + [("ONU", two)]:
            inp = ra.bound_inputs_for_plan(M, N, plan, 0.1)
            vals = [inp.prob_floor, inp.cancel_lo, inp.cancel_hi, inp.frob_m, inp.frob_n]
            vals += list(ra.bounds_optimal_allocation(inp))
            try:
                vals += list(ra.bounds_score_allocation(inp))
            except ValueError:  # pilot statistics outside [0, 1]: the reference refuses
                vals += [-1.0, -1.0]
            vals += list(ra.bounds_pilot_allocation(inp)) if inp.cancel_hi_exact is not None else [np.nan, np.nan]
            out[f"s{seed}_{meth}__bounds"] = np.array(vals)
            if meth == "ONU":
                out[f"s{seed}_ONU__budgets"] = plan.budgets
                out[f"s{seed}_ONU__pilot"] = plan.pilot_norms
    M, N, sizes, c, _ = sweep_params(NORMAL_SEED)
    part = ref.BlockPartition(sizes)
    plan = ref.allocate_optimal(M, N, part, c)
    res = ra.normality_diagnostic(M, N, plan, (1, 2), NORMAL_REPS, np.random.default_rng(9))
    out["normal__samples"] = res.samples
    out["normal__stats"] = np.array([res.mean, res.variance, res.ks_distance])
    np.savez_compressed(HERE / "analytics.npz", **out)


if __name__ == "__main__":
    main()
