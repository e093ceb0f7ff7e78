"""On-device instance generation (reference datagen.py:23-110):
the reference's own test strategy (tests/test_datagen.py there) -- validation,
hand-checked covariance, determinism per seed, target covariances and Cauchy
marginals -- since the device streams are distribution-identical, not
bit-identical, to numpy's."""
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


@pytest.mark.gpu
def test_shapes_determinism_and_errors():
    M, N = dg.gen_normal_instance(7, 50, 5, np.random.default_rng(3))
    assert M.shape == (7, 50) and N.shape == (50, 5) and M.dtype == np.float64
    M2, N2 = dg.gen_normal_instance(7, 50, 5, np.random.default_rng(3))
    assert np.array_equal(M, M2) and np.array_equal(N, N2)
    M3, _ = dg.gen_normal_instance(7, 50, 5, np.random.default_rng(4))
    assert not np.array_equal(M, M3)
    H, _ = dg.gen_heavy_tail_instance(7, 50, 5, np.random.default_rng(3))
    H2, _ = dg.gen_heavy_tail_instance(7, 50, 5, np.random.default_rng(3))
    assert np.array_equal(H, H2)
    Md, Nd = dg.gen_normal_instance(7, 50, 5, np.random.default_rng(3), device=True, dtype=np.float32)
    assert Md.is_cuda and Md.dtype == torch.float32 and np.allclose(Md.cpu().numpy(), M, rtol=1e-6, atol=1e-6)
    with pytest.raises(ValueError, match="dimensions"):
        dg.gen_normal_instance(0, 5, 5, np.random.default_rng(0))
    with pytest.raises(ValueError, match="location"):
        dg.gen_heavy_tail_instance(3, 5, 5, np.random.default_rng(0), location="half")
    with pytest.raises(ValueError, match="covariance dims"):
        dg.gen_normal_instance(3, 5, 5, np.random.default_rng(0), cov_left=dg.CovarianceSpec(4))


@pytest.mark.gpu
def test_normal_instance_matches_target_covariances():
    m, n, p = 6, 400000, 5
    left, right = dg.CovarianceSpec(m, 1.5, 0.6), dg.CovarianceSpec(p, 2.0, -0.4)
    M, N = dg.gen_normal_instance(m, n, p, np.random.default_rng(11), left, right)
    assert np.abs(M.mean(axis=1)).max() < 0.02 and np.abs(N.mean(axis=0)).max() < 0.02
    assert np.allclose(M @ M.T / n, dg.ar_covariance(left), atol=0.02)
    assert np.allclose(N.T @ N / n, dg.ar_covariance(right), atol=0.03)


@pytest.mark.gpu
def test_heavy_tail_cauchy_marginals():
    m, n, p = 4, 400000, 3
    M, N = dg.gen_heavy_tail_instance(m, n, p, np.random.default_rng(12))
    cl, cr = dg.ar_covariance(dg.CovarianceSpec(m, 1.0, 0.7)), dg.ar_covariance(dg.CovarianceSpec(p, 2.0, 0.7))
    # standard Cauchy quartiles are -1, 0, 1: |x - loc| / sqrt(Sigma_ii) has median 1
    for i in range(m):
        assert abs(np.median(np.abs(M[i] - 1.0)) / np.sqrt(cl[i, i]) - 1.0) < 0.02
    for f in range(p):
        assert abs(np.median(np.abs(N[:, f] - 1.0)) / np.sqrt(cr[f, f]) - 1.0) < 0.02
    Z, _ = dg.gen_heavy_tail_instance(m, 1000, p, np.random.default_rng(12), location="zero")
    Hn, _ = dg.gen_normal_instance(m, 1000, p, np.random.default_rng(12))
    assert np.abs(Z).max() > 10 * np.abs(Hn).max()  # heavier than normal
