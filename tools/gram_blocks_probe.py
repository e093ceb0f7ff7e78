"""Time bmm_segsq_gram (OPL g_k^2 by Gram matrices, DMMA) at config-4 and
config-5 shapes; prints ms and DMMA TF/s (executed: 36 of 64 tiles)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_04940_b200 import _lib  # noqa: E402


def run(name, B, m, n, p, L, reps=5):
    K = n // L
    M = torch.randn((B, m, n), dtype=torch.float32, device="cuda")
    N = torch.randn((B, n, p), dtype=torch.float32, device="cuda")
    off = torch.arange(0, n + 1, L, dtype=torch.int64, device="cuda")
    out = torch.empty(B * K, dtype=torch.float64, device="cuda")
    args = (_lib.BMM_F32, M.data_ptr(), n, m * n, N.data_ptr(), p, n * p, m, p, off.data_ptr(), K, 0, B,
            out.data_ptr(), _lib.stream_ptr())
    _lib.call("bmm_segsq_gram", *args)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("bmm_segsq_gram", *args)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    flops = 2.0 * (m + p) * n * L * 36 / 64 * B
    print(f"{name}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TF/s executed (DMMA)  "
          f"{4.0 * B * (m * n + n * p) / ms / 1e6:.0f} GB/s read", flush=True)
    del M, N
    torch.cuda.empty_cache()


if __name__ == "__main__":
    run("cfg5 (4096 x 256x4096x256, L=64)", 4096, 256, 4096, 256, 64)
    run("cfg4 (16384x262144x16384, L=64)", 1, 16384, 262144, 16384, 64, reps=3)
