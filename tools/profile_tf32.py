"""One large tcgen05 split-operand contraction (cfg4-like tile counts) for ncu:
m = p = 4096, K = 8192 float32 sketch columns.  Usage: python tools/profile_tf32.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_04940_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
m = p = 4096
K = 8192
g = torch.Generator(device="cuda").manual_seed(1)
a_hi = torch.randn(m * K, generator=g, device="cuda")
a_x = torch.randn(m * K, generator=g, device="cuda")
b_hi = torch.randn(p * K, generator=g, device="cuda")
b_x = torch.randn(p * K, generator=g, device="cuda")
out = torch.empty(m * p, device="cuda")
for _ in range(3):
    _lib.call("bmm_gemm_f32split", a_hi.data_ptr(), a_x.data_ptr(), b_hi.data_ptr(), b_x.data_ptr(), m, p, K, 1,
              out.data_ptr(), p, 0, _lib.stream_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_lib.call("bmm_gemm_f32split", a_hi.data_ptr(), a_x.data_ptr(), b_hi.data_ptr(), b_x.data_ptr(), m, p, K, 1,
          out.data_ptr(), p, 0, _lib.stream_ptr())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"{ms:.3f} ms, {2 * 2 * m * p * K / ms / 1e9:.0f} TF/s executed (2 MMAs per 8 K)")
