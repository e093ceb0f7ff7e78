"""Ozaki-scheme segmented square sums on the int8 tensor cores (bmm_segsq_i8)
against float64 references: the DMMA kernel (bmm_segsq_f64) and NumPy/OpenBLAS
(the reference's own arithmetic for g_k, plan.py:183-188).  Tolerance: 1e-13
relative per segment (float64 GEMMs themselves differ by ~1e-16-1e-15)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-13


def _np_gsq(M, N, seg):
    out = []
    for j in range(len(seg) - 1):
        P = M[:, seg[j]:seg[j + 1]] @ N[seg[j]:seg[j + 1], :]
        out.append(float(np.sum(P * P)))
    return np.array(out)


def _run(M, N, seg, n_inner=None, dtype=np.float64):
    from paper_2105_04940_b200 import _lib
    from paper_2105_04940_b200.plan import segsq_i8
    Md = torch.as_tensor(M.astype(dtype), device="cuda")
    Nd = torch.as_tensor(N.astype(dtype), device="cuda")
    s = _lib.i64(seg)
    return segsq_i8(Md, Nd, s, len(seg) - 1, n_inner).cpu().numpy()


def _check(got, ref, tol=TOL):
    ref = np.asarray(ref)
    scale = np.maximum(np.abs(ref), 1e-300)
    err = np.abs(got - ref) / scale
    err[ref == 0] = np.abs(got[ref == 0])
    assert np.all(np.isfinite(got))
    assert err.max() <= tol, f"max rel err {err.max():.3e} at {int(err.argmax())}"


@pytest.mark.parametrize("m,p", [(24, 16), (128, 64), (200, 200), (500, 500), (130, 70)])
def test_unequal_blocks(m, p):
    g = np.random.default_rng(11 + m + p)
    sizes = list(g.integers(1, 300, 23)) + [1, 32, 33, 64, 31]
    n = int(np.sum(sizes))
    seg = np.concatenate([[0], np.cumsum(sizes)])
    M = g.standard_normal((m, n)) * g.lognormal(0, 1, n)
    N = g.standard_normal((n, p)) * g.lognormal(0, 1, n)[:, None]
    _check(_run(M, N, seg), _np_gsq(M, N, seg))


def test_matches_dmma_kernel_cfg2_shape():
    from paper_2105_04940_b200 import _lib
    from paper_2105_04940_b200.plan import segsq
    g = np.random.default_rng(2)
    sizes = g.integers(100, 700, 50)
    n = int(sizes.sum())
    seg = np.concatenate([[0], np.cumsum(sizes)])
    M = g.standard_normal((500, n)) * g.lognormal(0, 1, n)
    N = g.standard_normal((n, 500)) * g.lognormal(0, 1, n)[:, None]
    got = _run(M, N, seg)
    dm = segsq(torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda"), _lib.i64(seg),
               len(sizes)).cpu().numpy()
    _check(got, dm)
    _check(got, _np_gsq(M, N, seg))


def test_zero_block_empty_segment_and_zero_rows():
    g = np.random.default_rng(5)
    sizes = [40, 0, 17, 64, 0, 90]
    n = sum(sizes)
    seg = np.concatenate([[0], np.cumsum(sizes)])
    M = g.standard_normal((70, n))
    N = g.standard_normal((n, 50))
    M[:, 57:121] = 0.0       # block 3 of M zero -> g = 0
    M[5, :] = 0.0            # a zero row
    N[:, 7] = 0.0            # a zero column
    got = _run(M, N, seg)
    ref = _np_gsq(M, N, seg)
    assert got[1] == 0.0 and got[4] == 0.0 and got[3] == 0.0
    _check(got, ref)


def test_wide_dynamic_range_and_float32():
    g = np.random.default_rng(8)
    sizes = [100, 250, 7, 300]
    n = sum(sizes)
    seg = np.concatenate([[0], np.cumsum(sizes)])
    M = g.standard_normal((96, n)) * np.exp(g.uniform(-20, 20, n))
    N = g.standard_normal((n, 80)) * np.exp(g.uniform(-20, 20, (n, 1)))
    _check(_run(M, N, seg), _np_gsq(M, N, seg), 1e-12)
    M32, N32 = M.astype(np.float32), N.astype(np.float32)
    _check(_run(M32, N32, seg, dtype=np.float32), _np_gsq(M32.astype(np.float64), N32.astype(np.float64), seg))


def test_offset_segments_and_many_segments():
    # segments starting mid-matrix (the streamed chunk calls), and > 1024 segments
    g = np.random.default_rng(9)
    sizes = g.integers(1, 12, 1500)
    n = int(sizes.sum()) + 37
    seg = 37 + np.concatenate([[0], np.cumsum(sizes)])
    M = g.standard_normal((40, n))
    N = g.standard_normal((n, 33))
    _check(_run(M, N, seg, n_inner=int(seg[-1] - seg[0])), _np_gsq(M, N, seg))


def test_deterministic():
    g = np.random.default_rng(3)
    sizes = g.integers(50, 400, 30)
    n = int(sizes.sum())
    seg = np.concatenate([[0], np.cumsum(sizes)])
    M = g.standard_normal((300, n))
    N = g.standard_normal((n, 260))
    a = _run(M, N, seg)
    b = _run(M, N, seg)
    assert np.array_equal(a, b)


def test_bad_segments_give_nan():
    g = np.random.default_rng(4)
    M = g.standard_normal((8, 100))
    N = g.standard_normal((100, 8))
    seg = np.array([0, 60, 40, 100])  # negative middle segment
    assert np.isnan(_run(M, N, seg)).all()
