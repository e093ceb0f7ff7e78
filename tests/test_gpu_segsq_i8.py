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


# ---- product mode: bmm_gemm_i8 / bmm_gemm_i8_gather (C @ D, estimators.py:175)

def _gemm_i8(A, B, k_dev=None, k_max=None, batch=1, kexp=None):
    from paper_2105_04940_b200 import _lib
    assert A.is_contiguous() and B.is_contiguous()
    dt = _lib.matrix_dtype(A)
    m, k = A.shape[-2:]
    p = B.shape[-1]
    k_max = k if k_max is None else k_max
    out = torch.empty((batch, m, p) if batch > 1 else (m, p), dtype=torch.float64, device="cuda")
    ws = _lib.workspace(_lib.load().bmm_gemm_i8_workspace(m, p, k_max, batch))
    _lib.call("bmm_gemm_i8", dt, A.data_ptr(), A.stride(-2), m * k if batch > 1 else 0, B.data_ptr(), B.stride(-2),
              k * p if batch > 1 else 0, m, p, k_max, k_dev.data_ptr() if k_dev is not None else None,
              kexp.data_ptr() if kexp is not None else None, batch,
              out.data_ptr(), p, m * p, ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    return out


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("m,k,p", [(1, 1, 1), (24, 100, 16), (500, 4400, 500), (130, 33, 70), (257, 9000, 129),
                                   (1000, 17000, 1000)])
def test_gemm_i8_matches_float64(m, k, p):
    g = np.random.default_rng(m + k + p)
    A = g.standard_normal((m, k)) * g.lognormal(0, 1.5, k)
    B = g.standard_normal((k, p)) * g.lognormal(0, 1.5, k)[:, None]
    Ad, Bd = torch.as_tensor(A, device="cuda"), torch.as_tensor(B, device="cuda")
    got = _gemm_i8(Ad, Bd).cpu().numpy()
    # one power-of-two scale per row / column over the whole inner length: 54-bit digits of
    # the largest entry, so heavy-tailed rows lose a few bits on their small entries (the
    # float64 pipeline's bar is 1e-12) ...
    assert _rel(got, A @ B) < 1e-12
    # ... unless the inner index is balanced (exact powers of two from the norms)
    from paper_2105_04940_b200 import _lib
    colsq = torch.as_tensor((A * A).sum(0), device="cuda")
    rowsq = torch.as_tensor((B * B).sum(1), device="cuda")
    kexp = torch.empty(k, dtype=torch.int32, device="cuda")
    _lib.call("bmm_balance_exponents", colsq.data_ptr(), rowsq.data_ptr(), 0, None, k, k, None, 1, kexp.data_ptr(),
              _lib.stream_ptr())
    got = _gemm_i8(Ad, Bd, kexp=kexp).cpu().numpy()
    assert _rel(got, A @ B) < 5e-14


def test_gemm_i8_device_length_batch_and_float32():
    from paper_2105_04940_b200 import _lib
    g = np.random.default_rng(7)
    bsz, m, k, p = 3, 200, 1000, 200
    A = g.standard_normal((bsz, m, k))
    B = g.standard_normal((bsz, k, p))
    kd = np.array([1000, 517, 0])
    got = _gemm_i8(torch.as_tensor(A, device="cuda"), torch.as_tensor(B, device="cuda"), k_dev=_lib.i64(kd),
                   batch=bsz).cpu().numpy()
    for b in range(bsz):
        ref = A[b, :, :kd[b]] @ B[b, :kd[b]]
        if kd[b] == 0:
            assert np.all(got[b] == 0)
        else:
            assert _rel(got[b], ref) < 1e-14
    A32, B32 = A[0].astype(np.float32), B[0].astype(np.float32)
    got = _gemm_i8(torch.as_tensor(A32, device="cuda"), torch.as_tensor(B32, device="cuda")).cpu().numpy()
    assert _rel(got, A32.astype(np.float64) @ B32.astype(np.float64)) < 1e-14


def test_gemm_i8_gather_matches_gathered_product():
    from paper_2105_04940_b200 import _lib
    g = np.random.default_rng(8)
    m, n, p, W = 150, 3000, 90, 777
    M = g.standard_normal((m, n)) * g.lognormal(0, 1, n)
    N = g.standard_normal((n, p))
    col = np.sort(g.choice(n, W, replace=False))
    sc = 1.0 / np.sqrt(g.uniform(0.01, 1.0, W) * 50)
    C = np.ascontiguousarray(M[:, col] * sc)
    D = np.ascontiguousarray(N[col, :] * sc[:, None])
    out = torch.empty((m, p), dtype=torch.float64, device="cuda")
    ws = _lib.workspace(_lib.load().bmm_gemm_i8_workspace(m, p, W, 1))
    kdev = _lib.i64([W - 5])
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    col_d, sc_d = _lib.i64(col), torch.as_tensor(sc, device="cuda")  # alive until the kernels ran
    _lib.call("bmm_gemm_i8_gather", 0, Md.data_ptr(), n, 0, Nd.data_ptr(), p, 0, col_d.data_ptr(),
              sc_d.data_ptr(), None, 0, m, p, W, kdev.data_ptr(), 1, out.data_ptr(), p, 0,
              ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    ref = C[:, :W - 5] @ D[:W - 5]
    assert _rel(out.cpu().numpy(), ref) < 1e-14
    # and bit-identical to the explicit-operand call on the gathered C, D
    out2 = _gemm_i8(torch.as_tensor(C, device="cuda"), torch.as_tensor(D, device="cuda"), k_dev=kdev)
    assert torch.equal(out, out2)
