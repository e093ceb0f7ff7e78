"""Golden outcomes of the reference on the randomised sweep instances
(tests/random_cases.py): for each seed and method, the budgets, drawn columns
and a product checksum -- or the exception class the reference raised.

Runs the REFERENCE package (``blockmm`` from /root/reference/pkg/src), so it
only works in the build container; the JSON output is committed.  Re-run with

    python tests/golden/make_random_sweep.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import blockmm as ref  # noqa: E402  (the reference, read-only)

from random_cases import random_instance, sweep_params  # noqa: E402

N_SEEDS = 40


def outcome(fn):
    try:
        plan, log, prod = fn()
    except AssertionError:
        return {"raises": "AssertionError"}
    except ValueError:
        return {"raises": "ValueError"}
    out = {"budgets": [int(x) for x in plan.budgets], "columns": [int(x) for x in log.column],
           "cd_sum": float(np.sum(prod)), "cd_norm": float(np.linalg.norm(prod))}
    if plan.pilot_norms is not None:
        out["pilot_norms"] = [float(x) for x in plan.pilot_norms]
    return out


def main():
    cases = []
    for seed in range(N_SEEDS):
        M, N, sizes, c, c0 = sweep_params(seed)
        part = ref.BlockPartition(sizes)
        res = {"seed": seed, "sizes": list(sizes), "c": c, "c0": c0}

        def one_step(alloc):
            plan = alloc(M, N, part, c)
            _, prod, log = ref.estimate_product(M, N, plan, np.random.default_rng(seed))
            return plan, log, prod

        def two_step(pilot):
            r = ref.estimate_product_two_step(M, N, part, c, c0, np.random.default_rng(seed), pilot=pilot)
            return r.plan, r.log, r.product

        res["ONC"] = outcome(lambda: one_step(ref.allocate_by_score_sums))
        res["OPL"] = outcome(lambda: one_step(ref.allocate_optimal))
        res["UU"] = outcome(lambda: one_step(lambda M_, N_, p_, c_: ref.allocate_uniform(p_, c_)))
        res["ONU"] = outcome(lambda: two_step("uniform"))
        res["ONMCNR"] = outcome(lambda: two_step("norm"))
        cases.append(res)
    (HERE / "random_sweep.json").write_text(json.dumps({"cases": cases}, indent=0))


if __name__ == "__main__":
    main()
