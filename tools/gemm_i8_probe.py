"""One bmm_gemm_i8 call per shape (for ncu launch lists): python tools/gemm_i8_probe.py m k p [reps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_04940_b200 import _lib  # noqa: E402

m, k, p = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn((m, k), generator=g, device="cuda", dtype=torch.float64)
B = torch.randn((k, p), generator=g, device="cuda", dtype=torch.float64)
O = torch.empty((m, p), dtype=torch.float64, device="cuda")
ws = _lib.workspace(_lib.load().bmm_gemm_i8_workspace(m, p, k, 1))
for _ in range(reps):
    _lib.call("bmm_gemm_i8", 0, A.data_ptr(), k, 0, B.data_ptr(), p, 0, m, p, k, None, None, 1, O.data_ptr(), p, 0,
              ws.data_ptr(), ws.numel(), _lib.stream_ptr())
torch.cuda.synchronize()
