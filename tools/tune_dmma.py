"""Time the DMMA tile variants on the shapes the hot path runs (cfg2 C.D and
OPL g_k, a square GEMM) and check they agree with variant 0."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import workloads  # noqa: E402
from paper_2105_04940_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
lib = _lib.load()
st = _lib.stream_ptr()
ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
shapes = [(500, 16000, 500), (500, 4000, 500), (1000, 20000, 1000), (4096, 4096, 4096), (256, 1024, 256)]
res = {}
for (m, k, n) in shapes:
    A = torch.randn(m, k, dtype=torch.float64, device="cuda")
    B = torch.randn(k, n, dtype=torch.float64, device="cuda")
    ref = None
    for v in range(7):
        lib.bmm_gemm_f64_set_variant(v, 0)
        out = torch.empty(m, n, dtype=torch.float64, device="cuda")
        f = lambda: lib.bmm_gemm_f64(A.data_ptr(), k, 0, B.data_ptr(), n, 0, m, n, k, 1, out.data_ptr(), n, 0,
                                     ws.data_ptr(), ws.numel(), st)
        for _ in range(3):
            f()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(10):
            f()
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 10
        if ref is None:
            ref = out.clone()
        err = ((out - ref).norm() / ref.norm()).item()
        print(f"gemm {m}x{k}x{n} v{v}: {ms*1e3:8.1f} us  {2*m*n*k/ms/1e9:6.2f} TF/s  diff {err:.1e}", flush=True)
# OPL segsq on cfg2
M, N, sizes = workloads.cfg2()
Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
off = torch.as_tensor(np.concatenate([[0], np.cumsum(sizes)]), device="cuda")
for v in range(7):
    lib.bmm_gemm_f64_set_variant(2, v)
    g = torch.empty(len(sizes), dtype=torch.float64, device="cuda")
    f = lambda: lib.bmm_segsq_f64(Md.data_ptr(), 20000, 0, Nd.data_ptr(), 500, 0, 500, 500, off.data_ptr(), len(sizes),
                                  0, 1, g.data_ptr(), ws.data_ptr(), ws.numel(), st)
    for _ in range(3):
        f()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        f()
    ev[1].record()
    torch.cuda.synchronize()
    print(f"segsq cfg2 v{v}: {ev[0].elapsed_time(ev[1]) / 10 * 1e3:8.1f} us", flush=True)
