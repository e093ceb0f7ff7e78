"""Instance generation (reference datagen.py:23-110).

stream="numpy" (default): the reference's own variates from the caller's Generator, the
Cholesky product on the device -- checked against instances written by the reference itself
(tests/golden/datagen.npz, tests/golden/make_datagen.py): every entry within 1e-13 of its
vector's norm (BLAS vs recursion rounding) and the generator left in the reference's state.
stream="device": the reference's own test strategy (tests/test_datagen.py there) --
validation, hand-checked covariance, determinism per seed, target covariances and Cauchy
marginals -- since the device streams are distribution-identical, not bit-identical, to
numpy's.  The statistical tests run on both modes."""
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
bm = pytest.importorskip("paper_2105_04940_b200")
from paper_2105_04940_b200 import datagen as dg  # noqa: E402


def test_covariance_spec_validation_and_hand_values():
    with pytest.raises(ValueError, match="dim"):
        dg.CovarianceSpec(0)
    with pytest.raises(ValueError, match="scale"):
        dg.CovarianceSpec(3, scale=0.0)
    with pytest.raises(ValueError, match="rho"):
        dg.CovarianceSpec(3, rho=1.0)
    c = dg.ar_covariance(dg.CovarianceSpec(3, scale=2.0, rho=0.5))
    assert np.array_equal(c, np.array([[2.0, 1.0, 0.5], [1.0, 2.0, 1.0], [0.5, 1.0, 2.0]]))


GOLDEN = Path(__file__).resolve().parent / "golden" / "datagen.npz"
# tests/golden/make_datagen.py CASES
CASES = [
    ("normal_default", False, 7, 50, 5, 3, None, None, None),
    ("normal_specs", False, 33, 301, 65, 11, (1.5, 0.6), (2.0, -0.4), None),
    ("normal_vec", False, 1, 9, 1, 5, (0.3, 0.0), (4.0, 0.95), None),
    ("heavy_ones", True, 7, 50, 5, 3, None, None, "ones"),
    ("heavy_zero", True, 40, 257, 31, 12, (1.0, -0.8), (0.5, 0.3), "zero"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_numpy_stream_matches_reference_instances(case):
    name, heavy, m, n, p, seed, left, right, loc = case
    g = np.load(GOLDEN)
    rng = np.random.default_rng(seed)
    cl = dg.CovarianceSpec(m, *left) if left else None
    cr = dg.CovarianceSpec(p, *right) if right else None
    if heavy:
        M, N = dg.gen_heavy_tail_instance(m, n, p, rng, cl, cr, location=loc)
    else:
        M, N = dg.gen_normal_instance(m, n, p, rng, cl, cr)
    # the caller's generator is left exactly where the reference leaves it
    assert np.array_equal(rng.bit_generator.random_raw(2), g[name + "_next"])
    Mr, Nr = g[name + "_M"], g[name + "_N"]
    assert M.shape == Mr.shape and N.shape == Nr.shape and M.dtype == np.float64 and N.flags.c_contiguous
    # tolerance: 1e-13 of the vector's norm (the reference's L @ Z is a BLAS product, ours the recursion)
    shift = (1.0 if loc == "ones" else 0.0)
    assert (np.abs(M - Mr).max(axis=0) <= 1e-13 * np.linalg.norm(Mr - shift, axis=0)).all()
    assert (np.abs(N - Nr).max(axis=1) <= 1e-13 * np.linalg.norm(Nr - shift, axis=1)).all()
    # float32 output: the same values rounded once
    rng = np.random.default_rng(seed)
    gen = dg.gen_heavy_tail_instance if heavy else dg.gen_normal_instance
    kw = {"location": loc} if heavy else {}
    M32, N32 = gen(m, n, p, rng, cl, cr, device=True, dtype=np.float32, **kw)
    assert M32.is_cuda and M32.dtype == torch.float32
    assert np.allclose(M32.cpu().numpy(), Mr.astype(np.float32), rtol=2e-6, atol=1e-6 * np.abs(Mr).max())
    assert np.allclose(N32.cpu().numpy(), Nr.astype(np.float32), rtol=2e-6, atol=1e-6 * np.abs(Nr).max())


@pytest.mark.gpu
@pytest.mark.parametrize("stream", ["numpy", "device"])
def test_shapes_determinism_and_errors(stream):
    M, N = dg.gen_normal_instance(7, 50, 5, np.random.default_rng(3), stream=stream)
    assert M.shape == (7, 50) and N.shape == (50, 5) and M.dtype == np.float64
    M2, N2 = dg.gen_normal_instance(7, 50, 5, np.random.default_rng(3), stream=stream)
    assert np.array_equal(M, M2) and np.array_equal(N, N2)
    M3, _ = dg.gen_normal_instance(7, 50, 5, np.random.default_rng(4), stream=stream)
    assert not np.array_equal(M, M3)
    H, _ = dg.gen_heavy_tail_instance(7, 50, 5, np.random.default_rng(3), stream=stream)
    H2, _ = dg.gen_heavy_tail_instance(7, 50, 5, np.random.default_rng(3), stream=stream)
    assert np.array_equal(H, H2)
    Md, Nd = dg.gen_normal_instance(7, 50, 5, np.random.default_rng(3), device=True, dtype=np.float32,
                                    stream=stream)
    assert Md.is_cuda and Md.dtype == torch.float32 and np.allclose(Md.cpu().numpy(), M, rtol=1e-6, atol=1e-6)
    with pytest.raises(ValueError, match="dimensions"):
        dg.gen_normal_instance(0, 5, 5, np.random.default_rng(0))
    with pytest.raises(ValueError, match="location"):
        dg.gen_heavy_tail_instance(3, 5, 5, np.random.default_rng(0), location="half")
    with pytest.raises(ValueError, match="covariance dims"):
        dg.gen_normal_instance(3, 5, 5, np.random.default_rng(0), cov_left=dg.CovarianceSpec(4))
    with pytest.raises(ValueError, match="stream"):
        dg.gen_normal_instance(3, 5, 5, np.random.default_rng(0), stream="other")


@pytest.mark.gpu
@pytest.mark.parametrize("stream", ["numpy", "device"])
def test_normal_instance_matches_target_covariances(stream):
    m, n, p = 6, 400000, 5
    left, right = dg.CovarianceSpec(m, 1.5, 0.6), dg.CovarianceSpec(p, 2.0, -0.4)
    M, N = dg.gen_normal_instance(m, n, p, np.random.default_rng(11), left, right, stream=stream)
    assert np.abs(M.mean(axis=1)).max() < 0.02 and np.abs(N.mean(axis=0)).max() < 0.02
    assert np.allclose(M @ M.T / n, dg.ar_covariance(left), atol=0.02)
    assert np.allclose(N.T @ N / n, dg.ar_covariance(right), atol=0.03)


@pytest.mark.gpu
@pytest.mark.parametrize("stream", ["numpy", "device"])
def test_heavy_tail_cauchy_marginals(stream):
    m, n, p = 4, 400000, 3
    M, N = dg.gen_heavy_tail_instance(m, n, p, np.random.default_rng(12), stream=stream)
    cl, cr = dg.ar_covariance(dg.CovarianceSpec(m, 1.0, 0.7)), dg.ar_covariance(dg.CovarianceSpec(p, 2.0, 0.7))
    # standard Cauchy quartiles are -1, 0, 1: |x - loc| / sqrt(Sigma_ii) has median 1
    for i in range(m):
        assert abs(np.median(np.abs(M[i] - 1.0)) / np.sqrt(cl[i, i]) - 1.0) < 0.02
    for f in range(p):
        assert abs(np.median(np.abs(N[:, f] - 1.0)) / np.sqrt(cr[f, f]) - 1.0) < 0.02
    Z, _ = dg.gen_heavy_tail_instance(m, 1000, p, np.random.default_rng(12), location="zero", stream=stream)
    Hn, _ = dg.gen_normal_instance(m, 1000, p, np.random.default_rng(12), stream=stream)
    assert np.abs(Z).max() > 10 * np.abs(Hn).max()  # heavier than normal
