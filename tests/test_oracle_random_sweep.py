"""Pin the oracle against the reference's own outcomes on the randomised sweep
(tests/golden/random_sweep.json, made by tests/golden/make_random_sweep.py):
zero columns, zero blocks, size-1 and very unequal blocks, every method --
including the cases where the reference raises (two-step plans whose
zero-weight hand-out drops a floor, plan.py:311-322 -> plan.py:146-152, and
non-converging apportionments, plan.py:306).  CPU only."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import blockmm_oracle as O
from random_cases import sweep_params

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "random_sweep.json").read_text())["cases"]


def outcome(fn):
    try:
        return fn()
    except AssertionError:
        return "AssertionError"
    except ValueError:
        return "ValueError"


@pytest.mark.parametrize("case", GOLD, ids=[f"seed{c['seed']}" for c in GOLD])
def test_oracle_matches_reference_sweep(case):
    seed = case["seed"]
    M, N, sizes, c, c0 = sweep_params(seed)
    assert list(sizes) == case["sizes"] and c == case["c"] and c0 == case["c0"]
    for meth in ("ONC", "OPL", "UU", "ONU", "ONMCNR"):
        want = case[meth]
        got = outcome(lambda: O.approx_product(M, N, sizes, c, meth, np.random.default_rng(seed), c0=c0))
        if "raises" in want:
            assert got == want["raises"], (seed, meth, got)
            continue
        assert not isinstance(got, str), (seed, meth, got)
        assert got["budgets"].tolist() == want["budgets"], (seed, meth)
        assert got["columns"].tolist() == want["columns"], (seed, meth)
        assert np.isclose(got["CD"].sum(), want["cd_sum"], rtol=1e-12, atol=1e-12 * want["cd_norm"])
        assert np.isclose(np.linalg.norm(got["CD"]), want["cd_norm"], rtol=1e-12, atol=0)
        if "pilot_norms" in want:
            assert np.allclose(np.sqrt(got["pilot_sq"]), want["pilot_norms"], rtol=1e-12, atol=0)
