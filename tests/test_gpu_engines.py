"""The int8 Ozaki engines forced on for every size (BMM_SEGSQ=i8 for the OPL
block-product norms, BMM_GEMM=i8 for the float64 sampled contraction; by
default they are chosen only for large problems): the randomised pipeline
sweep and the oracle-parity pipeline cases must hold unchanged -- indices,
budgets, probabilities and scales bit-exact, C.D within 1e-12 (float64) /
1e-5 (float32)."""
import numpy as np
import pytest

import test_gpu_pipeline
import test_gpu_random

pytestmark = pytest.mark.gpu


@pytest.fixture
def int8_engines(monkeypatch):
    monkeypatch.setenv("BMM_SEGSQ", "i8")
    monkeypatch.setenv("BMM_GEMM", "i8")


@pytest.mark.parametrize("seed", range(16))
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_random_pipeline_parity_int8(seed, dtype, int8_engines):
    test_gpu_random.test_random_pipeline_parity(seed, dtype)


@pytest.mark.parametrize("method", ["OPL", "ONC", "UU", "ONU", "ONMCNR"])
def test_pipeline_matches_oracle_int8(method, int8_engines):
    test_gpu_pipeline.test_pipeline_matches_oracle(method, True)


def test_engine_selection(monkeypatch):
    from paper_2105_04940_b200.plan import gemm_engine, segsq_engine
    monkeypatch.delenv("BMM_SEGSQ", raising=False)
    monkeypatch.delenv("BMM_GEMM", raising=False)
    assert segsq_engine(1000, 500, 500, 20000) == "i8"       # cfg2 OPL
    assert segsq_engine(100, 200, 200, 10000) == "dmma"      # cfg1: too small to pay for the split
    assert segsq_engine(40000, 500, 500, 100000) == "dmma"   # block beyond the exact int32 bound
    assert gemm_engine(1000, 1000, 20000) == "i8"            # cfg3 sketch
    assert gemm_engine(500, 500, 4000) == "dmma"
    monkeypatch.setenv("BMM_SEGSQ", "dmma")
    assert segsq_engine(1000, 500, 500, 20000) == "dmma"
