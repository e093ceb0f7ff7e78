import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
from test_gpu_tf32 import run_split_gemm
for (B, m, n, p, W) in [(2, 130, 777, 260, 4096), (1, 130, 777, 260, 4096), (1, 128, 777, 256, 4096), (1,128,777,128,8192), (2,128,777,128,1024)]:
    g = torch.Generator(device="cuda").manual_seed(5)
    M = torch.randn((B, m, n), generator=g, device="cuda", dtype=torch.float32)
    N = torch.randn((B, n, p), generator=g, device="cuda", dtype=torch.float32)
    column = torch.randint(0, n, (B, W), generator=g, device="cuda", dtype=torch.int64)
    scale = torch.rand((B, W), generator=g, device="cuda", dtype=torch.float64) * 3 + 0.1
    out, _ = run_split_gemm(M, N, column, scale, W)
    C64 = torch.gather(M.double(), 2, column[:, None, :].expand(B, m, W)) * scale[:, None, :]
    D64 = torch.gather(N.double(), 1, column[:, :, None].expand(B, W, p)) * scale[:, :, None]
    ref = torch.bmm(C64, D64)
    d = (out.double() - ref).abs()
    print((B,m,n,p,W), 'rel', ((out.double()-ref).norm()/ref.norm()).item())
    for b in range(B):
        for r0 in range(0, m, 128):
            for c0 in range(0, p, 128):
                blk = d[b, r0:r0+128, c0:c0+128]; rb = ref[b, r0:r0+128, c0:c0+128]
                print(f"  b{b} r{r0} c{c0}: maxabs {blk.max().item():.3e} rel {(blk.norm()/rb.norm()).item():.3e}")
    # one-pass estimate magnitude
