"""Time bmm_gemm_f32split_gather against the two-kernel split path on config-5
shaped problems (sorted compressed sketch columns, ~680 distinct of 4096).
Usage: python tools/fused_probe.py [B]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_04940_b200 import _lib  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
m = p = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 256
n, W, k = 4096, 1024, 680
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(1)
M = torch.randn((B, m, n), generator=g, device="cuda")
N = torch.randn((B, n, p), generator=g, device="cuda")
col = torch.sort(torch.rand((B, n), generator=g, device="cuda").argsort(dim=1)[:, :W], dim=1).values
col[:, k:] = 0
sc = torch.rand((B, W), generator=g, device="cuda", dtype=torch.float64) + 0.5
sc[:, k:] = 0
cnt = torch.full((B,), k, dtype=torch.int64, device="cuda")
out = torch.empty((B, m, p), device="cuda")
st = _lib.stream_ptr()
lib = _lib.load()
ahi = torch.empty((B * m, W), device="cuda")
ax = torch.empty((B * m, W), device="cuda")
bhi = torch.empty((B * p, W), device="cuda")
bx = torch.empty((B * p, W), device="cuda")
P = lambda t: t.data_ptr()  # noqa: E731
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def fused():
    _lib.call("bmm_gemm_f32split_gather", 1, P(M), n, m * n, P(N), p, n * p, m, p, P(col), P(sc), W, W, P(cnt), B,
              P(out), p, m * p, st)


def two():
    _lib.call("bmm_gather_f32split_dk", 1, P(M), n, m * n, P(N), p, n * p, m, p, P(col), P(sc), W, W, P(cnt), B,
              P(ahi), P(ax), P(bhi), P(bx), st)
    _lib.call("bmm_gemm_f32split_dk", P(ahi), P(ax), P(bhi), P(bx), m, p, W, P(cnt), B, P(out), p, m * p, st)


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


if "--once" in sys.argv:
    fused()
    torch.cuda.synchronize()
else:
    print(f"B={B}: fused {timed(fused):.3f} ms, two-kernel {timed(two):.3f} ms")
