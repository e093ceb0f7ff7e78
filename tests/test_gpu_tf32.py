"""float32 path: split gather + tcgen05 3xTF32 GEMM against a float64 reference
of the same sampled product (tolerance 1e-5 relative Frobenius, the north
star's float32 bar)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
from paper_2105_04940_b200 import _lib  # noqa: E402


def run_split_gemm(M, N, column, scale, W):
    B, m, n = M.shape
    p = N.shape[2]
    dev = M.device
    ahi = torch.empty((B * m, W), dtype=torch.float32, device=dev)
    alo = torch.empty_like(ahi)
    bhi = torch.empty((B * p, W), dtype=torch.float32, device=dev)
    blo = torch.empty_like(bhi)
    st = _lib.stream_ptr()
    _lib.call("bmm_gather_tf32x3", _lib.BMM_F32, M.data_ptr(), n, m * n, N.data_ptr(), p, n * p, m, p,
              column.data_ptr(), scale.data_ptr(), W, W, B, ahi.data_ptr(), alo.data_ptr(), bhi.data_ptr(),
              blo.data_ptr(), st)
    out = torch.empty((B, m, p), dtype=torch.float32, device=dev)
    _lib.call("bmm_gemm_tf32x3", ahi.data_ptr(), alo.data_ptr(), bhi.data_ptr(), blo.data_ptr(), m, p, W, B,
              out.data_ptr(), p, m * p, st)
    return out, (ahi, alo, bhi, blo)


@pytest.mark.parametrize("B,m,n,p,W", [(1, 128, 300, 128, 32), (1, 200, 2000, 72, 1000), (3, 256, 4096, 256, 1024),
                                       (2, 130, 777, 260, 4096), (1, 128, 64, 128, 4)])
def test_split_gather_and_tf32x3_gemm(B, m, n, p, W):
    g = torch.Generator(device="cuda").manual_seed(B * 1000 + m + n + p + W)
    M = torch.randn((B, m, n), generator=g, device="cuda", dtype=torch.float32)
    N = torch.randn((B, n, p), generator=g, device="cuda", dtype=torch.float32)
    column = torch.randint(0, n, (B, W), generator=g, device="cuda", dtype=torch.int64)
    scale = torch.rand((B, W), generator=g, device="cuda", dtype=torch.float64) * 3 + 0.1
    out, (ahi, alo, bhi, blo) = run_split_gemm(M, N, column, scale, W)
    torch.cuda.synchronize()
    # float64 reference of the same sketch
    idx = column
    C64 = torch.gather(M.double(), 2, idx[:, None, :].expand(B, m, W)) * scale[:, None, :]
    D64 = torch.gather(N.double(), 1, idx[:, :, None].expand(B, W, p)) * scale[:, :, None]
    ref = torch.bmm(C64, D64)
    # the split represents the float64 sketch to ~2^-24 relative
    rec = (ahi.double() + alo.double()).view(B, m, W)
    assert ((rec - C64).norm() / C64.norm()).item() < 1e-7
    err = ((out.double() - ref).norm() / ref.norm()).item()
    assert err < 1e-5, err
    # and it is genuinely better than a single TF32 pass would be
    one_pass = torch.bmm(ahi.view(B, m, W).double(), bhi.view(B, p, W).double().transpose(1, 2))
    assert err < ((one_pass - ref).norm() / ref.norm()).item()
