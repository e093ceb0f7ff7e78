"""float32 path: split gather + tcgen05 (TF32 leading products + BF16 cross
terms) GEMM against a float64 reference of the same sampled product
(tolerance 1e-5 relative Frobenius, the north star's float32 bar)."""
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
    ax = torch.empty((B * m, 2 * W), dtype=torch.bfloat16, device=dev)
    bhi = torch.empty((B * p, W), dtype=torch.float32, device=dev)
    bx = torch.empty((B * p, 2 * W), dtype=torch.bfloat16, device=dev)
    st = _lib.stream_ptr()
    _lib.call("bmm_gather_f32split", _lib.BMM_F32, M.data_ptr(), n, m * n, N.data_ptr(), p, n * p, m, p,
              column.data_ptr(), scale.data_ptr(), W, W, B, ahi.data_ptr(), ax.data_ptr(), bhi.data_ptr(),
              bx.data_ptr(), st)
    out = torch.empty((B, m, p), dtype=torch.float32, device=dev)
    _lib.call("bmm_gemm_f32split", ahi.data_ptr(), ax.data_ptr(), bhi.data_ptr(), bx.data_ptr(), m, p, W, B,
              out.data_ptr(), p, m * p, st)
    return out, (ahi, ax, bhi, bx)


def unpair(x, W, first):
    """(rows, 2W) bf16 pair rows -> the (rows, W) half at offset 0 (first) or 8."""
    g = x.view(x.shape[0], W // 8, 16)
    return (g[:, :, :8] if first else g[:, :, 8:]).reshape(x.shape[0], W).double()


@pytest.mark.parametrize("B,m,n,p,W", [(1, 128, 300, 128, 32), (1, 200, 2000, 72, 1000), (3, 256, 4096, 256, 1024),
                                       (2, 130, 777, 260, 4096), (1, 128, 64, 128, 8), (1, 128, 999, 128, 32768),
                                       (2, 384, 1500, 640, 512), (1, 256, 3000, 1024, 2048),
                                       # cta_group::2 (256 x 256 pair tiles): partial pair tiles, long K
                                       (1, 300, 2000, 520, 1024), (1, 512, 5000, 768, 4096),
                                       (1, 256, 999, 512, 32768), (3, 260, 700, 1030, 256)])
def test_split_gather_and_gemm(B, m, n, p, W):
    g = torch.Generator(device="cuda").manual_seed(B * 1000 + m + n + p + W)
    M = torch.randn((B, m, n), generator=g, device="cuda", dtype=torch.float32)
    N = torch.randn((B, n, p), generator=g, device="cuda", dtype=torch.float32)
    column = torch.randint(0, n, (B, W), generator=g, device="cuda", dtype=torch.int64)
    scale = torch.rand((B, W), generator=g, device="cuda", dtype=torch.float64) * 3 + 0.1
    out, (ahi, ax, bhi, bx) = run_split_gemm(M, N, column, scale, W)
    torch.cuda.synchronize()
    C64 = torch.gather(M.double(), 2, column[:, None, :].expand(B, m, W)) * scale[:, None, :]
    D64 = torch.gather(N.double(), 1, column[:, :, None].expand(B, W, p)) * scale[:, :, None]
    ref = torch.bmm(C64, D64)
    # operand layout: tf32 hi exactly tf32-rounded; bf16 pairs [h|l] for A, [l|h] for D^T
    hi = ahi.view(B, m, W).double()
    assert ((hi - C64).norm() / C64.norm()).item() < 2 ** -10
    lo_a = unpair(ax, W, first=False).view(B, m, W)
    assert ((hi + lo_a - C64).norm() / C64.norm()).item() < 1e-5
    hi_d = bhi.view(B, p, W).double().transpose(1, 2)
    lo_d = unpair(bx, W, first=True).view(B, p, W).transpose(1, 2)
    assert ((hi_d + lo_d - D64).norm() / D64.norm()).item() < 1e-5
    err = ((out.double() - ref).norm() / ref.norm()).item()
    assert err < 1e-5, err
    # and it is genuinely better than a single TF32 pass would be
    one_pass = torch.bmm(hi, hi_d)
    assert err < 0.1 * ((one_pass - ref).norm() / ref.norm()).item()


def test_cta_pair_multicast_variant_matches():
    """The opt-in CTA-pair (TMA multicast) contraction, run in a fresh process with
    BMM_TF32_PAIR=1, gives bit-identical products to the default single-CTA one
    (same MMAs per tile, same accumulation order)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    code = (
        "import torch, numpy as np, sys\n"
        "sys.path[:0] = [%r, %r]\n"
        "from test_gpu_tf32 import run_split_gemm\n"
        "g = torch.Generator(device='cuda').manual_seed(5)\n"
        "M = torch.randn((2, 384, 1500), generator=g, device='cuda')\n"
        "N = torch.randn((2, 1500, 640), generator=g, device='cuda')\n"
        "col = torch.randint(0, 1500, (2, 512), generator=g, device='cuda')\n"
        "sc = torch.rand((2, 512), generator=g, device='cuda', dtype=torch.float64) + 0.5\n"
        "out, _ = run_split_gemm(M, N, col, sc, 512)\n"
        "np.save(sys.argv[1], out.cpu().numpy())\n" % (str(Path(__file__).resolve().parent),
                                                         str(Path(__file__).resolve().parent.parent)))
    outs = []
    for pair in ("0", "1"):
        f = Path(os.environ.get("TMPDIR", "/tmp")) / f"bmm_pair_{pair}_{os.getpid()}.npy"
        env = dict(os.environ, BMM_TF32_PAIR=pair)
        subprocess.run([sys.executable, "-c", code, str(f)], env=env, check=True, timeout=300)
        outs.append(np.load(f))
        f.unlink()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("B,m,n,p,W", [(3, 256, 4096, 256, 1024), (2, 130, 777, 260, 512), (1, 200, 2000, 72, 1000),
                                       (4, 128, 300, 128, 32), (1, 512, 3000, 512, 4096), (2, 64, 500, 200, 200)])
def test_fused_gather_gemm(B, m, n, p, W):
    """bmm_gemm_f32split_gather (the split gather inside the contraction's producer
    warps) against the float64 product of the same sketch prefix (first count[b]
    columns; one problem with count 0), and against the two-kernel path."""
    g = torch.Generator(device="cuda").manual_seed(7 * B + m + n + p + W)
    M = torch.randn((B, m, n), generator=g, device="cuda", dtype=torch.float32)
    N = torch.randn((B, n, p), generator=g, device="cuda", dtype=torch.float32)
    column = torch.sort(torch.randint(0, n, (B, W), generator=g, device="cuda", dtype=torch.int64), dim=1).values
    scale = torch.rand((B, W), generator=g, device="cuda", dtype=torch.float64) * 3 + 0.1
    count = torch.randint(W // 2, W + 1, (B,), generator=g, device="cuda", dtype=torch.int64)
    count[0] = W
    if B > 2:
        count[1] = 0
    out = torch.full((B, m, p), float("nan"), dtype=torch.float32, device="cuda")
    _lib.call("bmm_gemm_f32split_gather", _lib.BMM_F32, M.data_ptr(), n, m * n, N.data_ptr(), p, n * p, m, p,
              column.data_ptr(), scale.data_ptr(), W, W, count.data_ptr(), B, out.data_ptr(), p, m * p,
              _lib.stream_ptr())
    torch.cuda.synchronize()
    C64 = torch.gather(M.double(), 2, column[:, None, :].expand(B, m, W)) * scale[:, None, :]
    D64 = torch.gather(N.double(), 1, column[:, :, None].expand(B, W, p)) * scale[:, :, None]
    keep = (torch.arange(W, device="cuda")[None, :] < count[:, None]).double()
    ref = torch.bmm(C64 * keep[:, None, :], D64)
    assert torch.isfinite(out).all()
    for b in range(B):
        if int(count[b]) == 0:
            assert (out[b] == 0).all()
            continue
        err = ((out[b].double() - ref[b]).norm() / ref[b].norm()).item()
        assert err < 1e-5, (b, err)
    # without counts: all W columns, close to the two-kernel path on the same sketch
    if W % 8 == 0:
        _lib.call("bmm_gemm_f32split_gather", _lib.BMM_F32, M.data_ptr(), n, m * n, N.data_ptr(), p, n * p, m, p,
                  column.data_ptr(), scale.data_ptr(), W, W, None, B, out.data_ptr(), p, m * p, _lib.stream_ptr())
        two, _ = run_split_gemm(M, N, column, scale, W)
        full = torch.bmm(C64, D64)
        torch.cuda.synchronize()
        e_fused = ((out.double() - full).norm() / full.norm()).item()
        e_two = ((two.double() - full).norm() / full.norm()).item()
        assert e_fused < 1e-5 and e_two < 1e-5, (e_fused, e_two)


@pytest.mark.parametrize("B,m,p,n,W,spread", [(1, 256, 512, 3000, 1024, 1.0), (2, 300, 520, 2000, 2048, 4.0),
                                              (1, 512, 768, 5000, 4096, 8.0), (1, 256, 1024, 999, 32768, 2.0)])
def test_f16_split_pair_contraction(B, m, p, n, W, spread):
    """The fp16 split on CTA pairs (bmm_balance_f16 + bmm_gather_f16split_dk +
    bmm_gemm_f16split_dk) on compressed sketches: distinct counts not a multiple
    of 64, a zero column, lognormal column / row scales of wide spread (the
    balanced exponents and the shift must keep both operands in fp16 range),
    partial pair tiles and batches -- against float64 of the same float32 sketch
    (C = fl32(M * s), D = fl32(N * s)) within 1e-5."""
    g = torch.Generator(device="cuda").manual_seed(B * 7 + m + p + W)
    M = torch.randn((B, m, n), generator=g, device="cuda") * torch.exp(spread * torch.randn((B, 1, n), generator=g, device="cuda"))
    N = torch.randn((B, n, p), generator=g, device="cuda") * torch.exp(spread * torch.randn((B, n, 1), generator=g, device="cuda"))
    M[:, :, 3] = 0.0  # a zero column of M
    colsq = (M.double() ** 2).sum(1).reshape(-1)
    rowsq = (N.double() ** 2).sum(2).reshape(-1)
    cnt = [min(W, n, 1000 + 37 * b + (W // 3)) for b in range(B)]
    col = torch.zeros((B, W), dtype=torch.int64, device="cuda")
    sc = torch.zeros((B, W), dtype=torch.float64, device="cuda")
    for b in range(B):
        c = torch.sort(torch.randperm(n, generator=g, device="cuda")[:cnt[b]]).values
        col[b, :cnt[b]] = c
        sc[b, :cnt[b]] = torch.rand(cnt[b], generator=g, device="cuda", dtype=torch.float64) * 50 + 0.01
    kd = torch.as_tensor(cnt, dtype=torch.int64, device="cuda")
    kexp = torch.zeros((B, W), dtype=torch.int32, device="cuda")
    gsh = torch.zeros(B, dtype=torch.int32, device="cuda")
    st = _lib.stream_ptr()
    _lib.call("bmm_balance_f16", colsq.data_ptr(), rowsq.data_ptr(), n, col.data_ptr(), sc.data_ptr(), W, W,
              kd.data_ptr(), B, kexp.data_ptr(), gsh.data_ptr(), st)
    ah = torch.full((B * m * W,), float("nan"), dtype=torch.float32, device="cuda")  # garbage past the K step
    ax = torch.full_like(ah, float("nan"))
    bh = torch.full((B * p * W,), float("nan"), dtype=torch.float32, device="cuda")
    bx = torch.full_like(bh, float("nan"))
    _lib.call("bmm_gather_f16split_dk", _lib.BMM_F32, M.data_ptr(), n, m * n, N.data_ptr(), p, n * p, m, p,
              col.data_ptr(), sc.data_ptr(), kexp.data_ptr(), gsh.data_ptr(), W, W, kd.data_ptr(), B,
              ah.data_ptr(), ax.data_ptr(), bh.data_ptr(), bx.data_ptr(), st)
    out = torch.empty((B, m, p), dtype=torch.float32, device="cuda")
    _lib.call("bmm_gemm_f16split_dk", ah.data_ptr(), ax.data_ptr(), bh.data_ptr(), bx.data_ptr(), m, p, W,
              kd.data_ptr(), gsh.data_ptr(), B, out.data_ptr(), p, m * p, st)
    torch.cuda.synchronize()
    for b in range(B):
        c, s = col[b, :cnt[b]], sc[b, :cnt[b]]
        C = (M[b][:, c] * s.float()).double()          # the float32 sketch values
        D = (N[b][c, :] * s.float()[:, None]).double()
        ref = C @ D
        err = ((out[b].double() - ref).norm() / ref.norm()).item()
        assert err < 1e-5, (b, err)
        assert torch.isfinite(out[b]).all()


@pytest.mark.parametrize("B,m,p,n,W,spread,zero", [
    (3, 256, 256, 4096, 1024, 0.5, False),   # config-5 shape
    (2, 200, 252, 2048, 512, 2.0, False),    # ragged rows / columns inside one tile
    (2, 300, 140, 1500, 1000, 1.0, False),   # two row tiles, one column tile
    (2, 256, 256, 1024, 96, 0.5, True),      # a problem with no drawn column (count 0)
])
def test_f16_split_fused_gather(B, m, p, n, W, spread, zero):
    """bmm_gemm_f16split_gather (gather + fp16 split + contraction in one kernel,
    one CTA per 256 x 256 tile): distinct counts not a multiple of 32, a zero
    column, wide column / row scales, ragged tiles and an empty sketch -- against
    float64 of the same float32 sketch within 1e-5."""
    g = torch.Generator(device="cuda").manual_seed(B * 11 + m + p + W)
    M = torch.randn((B, m, n), generator=g, device="cuda") * torch.exp(spread * torch.randn((B, 1, n), generator=g, device="cuda"))
    N = torch.randn((B, n, p), generator=g, device="cuda") * torch.exp(spread * torch.randn((B, n, 1), generator=g, device="cuda"))
    M[:, :, 3] = 0.0
    colsq = (M.double() ** 2).sum(1).reshape(-1)
    rowsq = (N.double() ** 2).sum(2).reshape(-1)
    cnt = [min(W, n, (W * 2) // 3 + 37 * b + 5) for b in range(B)]
    if zero:
        cnt[0] = 0
    col = torch.zeros((B, W), dtype=torch.int64, device="cuda")
    sc = torch.zeros((B, W), dtype=torch.float64, device="cuda")
    for b in range(B):
        c = torch.sort(torch.randperm(n, generator=g, device="cuda")[:cnt[b]]).values
        col[b, :cnt[b]] = c
        sc[b, :cnt[b]] = torch.rand(cnt[b], generator=g, device="cuda", dtype=torch.float64) * 50 + 0.01
    kd = torch.as_tensor(cnt, dtype=torch.int64, device="cuda")
    kexp = torch.zeros((B, W), dtype=torch.int32, device="cuda")
    gsh = torch.zeros(B, dtype=torch.int32, device="cuda")
    st = _lib.stream_ptr()
    _lib.call("bmm_balance_f16", colsq.data_ptr(), rowsq.data_ptr(), n, col.data_ptr(), sc.data_ptr(), W, W,
              kd.data_ptr(), B, kexp.data_ptr(), gsh.data_ptr(), st)
    out = torch.full((B, m, p), float("nan"), dtype=torch.float32, device="cuda")
    _lib.call("bmm_gemm_f16split_gather", _lib.BMM_F32, M.data_ptr(), n, m * n, N.data_ptr(), p, n * p, m, n, p,
              col.data_ptr(), sc.data_ptr(), kexp.data_ptr(), gsh.data_ptr(), W, W, kd.data_ptr(), B,
              out.data_ptr(), p, m * p, st)
    torch.cuda.synchronize()
    for b in range(B):
        assert torch.isfinite(out[b]).all(), b
        if cnt[b] == 0:
            assert (out[b] == 0).all()
            continue
        c, s = col[b, :cnt[b]], sc[b, :cnt[b]]
        C = (M[b][:, c] * s.float()).double()
        D = (N[b][c, :] * s.float()[:, None]).double()
        ref = C @ D
        err = ((out[b].double() - ref).norm() / ref.norm()).item()
        assert err < 1e-5, (b, err)
    # rows of N that TMA cannot address (p % 4 != 0) are refused, not misread
    if p % 8 == 4:
        with pytest.raises(RuntimeError, match="16-byte aligned"):
            _lib.call("bmm_gemm_f16split_gather", _lib.BMM_F32, M.data_ptr(), n, m * n, N.data_ptr(), p - 2,
                      n * p, m, n, p - 2, col.data_ptr(), sc.data_ptr(), kexp.data_ptr(), gsh.data_ptr(), W, W,
                      kd.data_ptr(), B, out.data_ptr(), p, m * p, st)
    # the float32 path's dtype check: float64 inputs are refused, not misread
    with pytest.raises(RuntimeError):
        _lib.call("bmm_gemm_f16split_gather", _lib.BMM_F64, M.data_ptr(), n, m * n, N.data_ptr(), p, n * p, m, n, p,
                  col.data_ptr(), sc.data_ptr(), kexp.data_ptr(), gsh.data_ptr(), W, W, kd.data_ptr(), B,
                  out.data_ptr(), p, m * p, st)
