"""Time bmm_segsq_i8 against the DMMA bmm_segsq_f64 on the cfg2 / cfg3 OPL
shapes (CUDA events, warm, L2 not flushed) and report the agreement.
Usage: python tools/segsq_i8_bench.py [gemm]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import workloads  # noqa: E402
from paper_2105_04940_b200 import _lib  # noqa: E402

lib = _lib.load()


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for name in (() if "gemm" in sys.argv else ("cfg2", "cfg3", "cfg1")):
    M, N, sizes = getattr(workloads, name)()[:3]
    M = torch.as_tensor(M, device="cuda")
    N = torch.as_tensor(N, device="cuda")
    m, n = M.shape
    p = N.shape[1]
    K = len(sizes)
    seg = _lib.i64(np.concatenate([[0], np.cumsum(sizes)]))
    g8 = torch.empty(K, dtype=torch.float64, device="cuda")
    g64 = torch.empty(K, dtype=torch.float64, device="cuda")
    w8 = _lib.workspace(lib.bmm_segsq_i8_workspace(m, p, n, K, 1))
    w64 = _lib.workspace(lib.bmm_segsq_f64_workspace(m, p, K, 1))
    st = _lib.stream_ptr()
    f8 = lambda: _lib.call("bmm_segsq_i8", 0, M.data_ptr(), n, 0, N.data_ptr(), p, 0, m, p, n, seg.data_ptr(), K, 0, 1,
                           g8.data_ptr(), w8.data_ptr(), w8.numel(), st)
    f64 = lambda: _lib.call("bmm_segsq_f64", M.data_ptr(), n, 0, N.data_ptr(), p, 0, m, p, seg.data_ptr(), K, 0, 1,
                            g64.data_ptr(), w64.data_ptr(), w64.numel(), st)
    t8, t64 = timeit(f8), timeit(f64)
    rel = (g8 - g64).abs().max().item() / g64.abs().max().item()
    relmax = ((g8 - g64).abs() / g64.abs()).max().item()
    flops = 2.0 * m * p * n
    print(f"{name}: m={m} n={n} p={p} K={K}  i8 {t8*1e3:8.1f} us ({flops/t8/1e9:6.1f} TF/s f64-equiv)  "
          f"dmma {t64*1e3:8.1f} us ({flops/t64/1e9:6.1f} TF/s)  rel diff max {relmax:.2e}", flush=True)

# ---- sampled-GEMM shapes: bmm_gemm_i8 vs bmm_gemm_f64 (DMMA)
for (m, k, p) in ((500, 1900, 500), (500, 4400, 500), (1000, 17000, 1000), (200, 2000, 200)):
    g = np.random.default_rng(1)
    A = torch.as_tensor(g.standard_normal((m, k)), device="cuda")
    B = torch.as_tensor(g.standard_normal((k, p)), device="cuda")
    o8 = torch.empty((m, p), dtype=torch.float64, device="cuda")
    o64 = torch.empty((m, p), dtype=torch.float64, device="cuda")
    w8 = _lib.workspace(lib.bmm_gemm_i8_workspace(m, p, k, 1))
    w64 = _lib.workspace(lib.bmm_gemm_f64_workspace(m, p, k, 1))
    st = _lib.stream_ptr()
    f8 = lambda: _lib.call("bmm_gemm_i8", 0, A.data_ptr(), k, 0, B.data_ptr(), p, 0, m, p, k, None, None, 1, o8.data_ptr(),
                           p, 0, w8.data_ptr(), w8.numel(), st)
    f64 = lambda: _lib.call("bmm_gemm_f64", A.data_ptr(), k, 0, B.data_ptr(), p, 0, m, p, k, 1, o64.data_ptr(), p, 0,
                            w64.data_ptr(), w64.numel(), st)
    t8, t64 = timeit(f8), timeit(f64)
    rel = ((o8 - o64).norm() / o64.norm()).item()
    flops = 2.0 * m * p * k
    print(f"gemm {m}x{k}x{p}: i8 {t8*1e3:8.1f} us ({flops/t8/1e9:6.1f} TF/s f64-equiv)  dmma {t64*1e3:8.1f} us "
          f"({flops/t64/1e9:6.1f} TF/s)  rel diff {rel:.2e}", flush=True)
