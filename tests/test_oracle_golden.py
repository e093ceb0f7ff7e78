"""Pin the CPU oracle (oracle/blockmm_oracle.py) against golden vectors made
by running the reference itself (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

import workloads
from oracle import blockmm_oracle as O
from golden_cases import make_instance, ssm_draws


def _cases(meta):
    return [pytest.param(c, id=c["name"]) for c in meta["cases"]]


def test_small_cases_bit_exact(golden_meta, golden_small):
    for case in golden_meta["cases"]:
        M, N = make_instance(case)
        g = {k.split("__", 1)[1]: v for k, v in golden_small.items() if k.startswith(case["name"] + "__")}
        sizes, c, c0 = case["sizes"], case["c"], case["c0"]
        cs, rs, probs, s = O.instance_stats(M, N, sizes)
        assert np.array_equal(np.sqrt(cs), g["colnorm"])
        assert np.array_equal(np.sqrt(rs), g["rownorm"])
        assert np.array_equal(s, g["s"])
        assert np.array_equal(probs, g["probs"])
        for meth in ("OPL", "ONC", "UU"):
            res = O.approx_product(M, N, sizes, c, meth, np.random.default_rng(case["sample_seed"]))
            assert np.array_equal(res["budgets"], g[f"{meth}_budgets"]), (case["name"], meth)
            assert np.array_equal(res["columns"], g[f"{meth}_columns"]), (case["name"], meth)
            if meth != "UU":
                assert np.array_equal(res["scale"], g[f"{meth}_scale"])
            np.testing.assert_allclose(res["CD"], g[f"{meth}_CD"], rtol=1e-12, atol=1e-12)
        for meth in ("ONU", "ONMCNR"):
            res = O.approx_product(M, N, sizes, c, meth, np.random.default_rng(case["sample_seed"]), c0=c0)
            assert np.array_equal(res["budgets"], g[f"{meth}_budgets"]), (case["name"], meth)
            np.testing.assert_allclose(np.sqrt(res["pilot_sq"]), g[f"{meth}_pilot"], rtol=1e-12)
            assert np.array_equal(res["columns"], g[f"{meth}_columns"])
            np.testing.assert_allclose(res["CD"], g[f"{meth}_CD"], rtol=1e-12, atol=1e-12)
        res = O.ssm_product(M, N, sizes, ssm_draws(case), np.random.default_rng(case["sample_seed"]))
        np.testing.assert_allclose(res["q"], g["SSM_q"], rtol=1e-14)
        assert np.array_equal(res["blocks"], g["SSM_blocks"])
        np.testing.assert_allclose(res["scale"], g["SSM_scale"], rtol=1e-14)
        np.testing.assert_allclose(res["CD"], g["SSM_CD"], rtol=1e-12, atol=1e-12)


def test_cfg1_bit_exact(golden_cfg1):
    M, N, sizes = workloads.cfg1()
    g = golden_cfg1
    cs, rs, probs, s = O.instance_stats(M, N, sizes)
    assert np.array_equal(probs, g["probs"])
    assert np.array_equal(s, g["s"])
    for meth in ("OPL", "ONC"):
        res = O.approx_product(M, N, sizes, 2000, meth, workloads.sample_rng(1))
        assert np.array_equal(res["budgets"], g[f"{meth}_budgets"])
        assert np.array_equal(res["columns"], g[f"{meth}_columns"])
        assert np.array_equal(res["scale"], g[f"{meth}_scale"])
        np.testing.assert_allclose(res["CD"], g[f"{meth}_CD"], rtol=1e-12, atol=1e-11)
    res = O.ssm_product(M, N, sizes, 20, workloads.sample_rng(1))
    assert np.array_equal(res["blocks"], g["SSM_blocks"])


def test_cfg2_bit_exact(golden_cfg2):
    M, N, sizes = workloads.cfg2()
    g = golden_cfg2
    assert tuple(g["sizes"]) == sizes
    for c_blocks, W in zip((10, 20, 40), (4000, 8000, 16000)):
        for meth in ("OPL", "ONC", "ONMCNR"):
            res = O.approx_product(M, N, sizes, W, meth, workloads.sample_rng(2, c_blocks), c0=500)
            assert np.array_equal(res["budgets"], g[f"{meth}_{W}_budgets"]), (meth, W)
            assert np.array_equal(res["columns"], g[f"{meth}_{W}_columns"]), (meth, W)
            assert np.array_equal(res["scale"], g[f"{meth}_{W}_scale"])
            np.testing.assert_allclose(res["CD"][::7, ::7], g[f"{meth}_{W}_CDsub"], rtol=1e-10, atol=1e-9)


def test_integerize_known_answers(golden_meta):
    for case in golden_meta["integerize"]:
        w = np.array(case["w"])
        caps = None if case["caps"] is None else np.array(case["caps"])
        floors = None if case["floors"] is None else np.array(case["floors"])
        if case["err"] == "ValueError":
            with pytest.raises(ValueError):
                O.integerize(w, case["c"], caps, floors)
        elif case["err"] == "AssertionError":
            with pytest.raises(AssertionError):
                O.integerize(w, case["c"], caps, floors)
        else:
            assert O.integerize(w, case["c"], caps, floors).tolist() == case["out"]
