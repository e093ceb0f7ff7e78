"""Small instances that launch every hot kernel once, for compute-sanitizer
(memcheck / racecheck / synccheck):  python tools/sanitize_kernels.py [part]
parts: f32 (norms: colsq_vec + rowsq_tma, block probabilities, budgets, sampling,
compaction, split gather + tcgen05 contraction, fused gather-contraction, SSM
expansion, Gram g_k), f64 (colsq/rowsq TMA/leaf kernels, int8 Ozaki g_k and
C.D, DMMA GEMM, two-step Gram pilot), wide (the TMA one-wave colsq, forced on a
small matrix).  Each part checks its result against the pipeline's own
invariants only; parity is the tests' job."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import workloads  # noqa: E402
from paper_2105_04940_b200 import _lib  # noqa: E402
from paper_2105_04940_b200.pipeline import PipelineGroup, SketchPipeline, seeds_from_keys, seeds_from_rngs  # noqa: E402

torch.cuda.set_device(0)
part = sys.argv[1] if len(sys.argv) > 1 else "all"


def f32():
    g = torch.Generator(device="cuda").manual_seed(3)
    B, m, n, p, K = 2, 256, 4096, 256, 64
    M = torch.randn((B, m, n), generator=g, device="cuda")
    N = torch.randn((B, n, p), generator=g, device="cuda")
    for fused in ("0", "1"):
        os.environ["BMM_F32_FUSED"] = fused
        pipe = SketchPipeline(m, n, p, (64,) * K, 1024, "ONC", batch=B, dtype=torch.float32)
        pipe.run(M, N, seeds_from_keys("ONC", workloads.ROOT, (5, 1), np.arange(B), K))
        pipe.check()
    os.environ.pop("BMM_F32_FUSED")
    # one instance: OPL (Gram g_k) + ONC + SSM sharing statistics, 128x128 split contraction
    M1, N1 = M[0].contiguous(), N[0].contiguous()
    grp = PipelineGroup([SketchPipeline(m, n, p, (64,) * K, 512, "OPL", dtype=torch.float32),
                         SketchPipeline(m, n, p, (64,) * K, 512, "ONC", dtype=torch.float32),
                         SketchPipeline(m, n, p, (64,) * K, 0, "SSM", draws=6, dtype=torch.float32)])
    grp.run(M1, N1, [seeds_from_rngs("OPL", [np.random.default_rng(1)], K),
                     seeds_from_rngs("ONC", [np.random.default_rng(2)], K),
                     seeds_from_rngs("SSM", [np.random.default_rng(3)], K, draws=6)])
    grp.check()


def f64():
    M, N, sizes = workloads.cfg2(n=4000, m=128, p=96, K=12)
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    for seg, gemm in (("i8", "i8"), ("dmma", "dmma")):
        os.environ["BMM_SEGSQ"], os.environ["BMM_GEMM"] = seg, gemm
        for meth in ("OPL", "ONU"):
            pipe = SketchPipeline(128, 4000, 96, sizes, 1200, meth, c0=60)
            pipe.run(Md, Nd, seeds_from_rngs(meth, [np.random.default_rng(4)], len(sizes)))
            pipe.check()
    for k in ("BMM_SEGSQ", "BMM_GEMM"):
        os.environ.pop(k)


def wide():  # run with BMM_COLSQ_WIDE=2 (read once per process by csrc/norms.cu)
    for dt in (torch.float32, torch.float64):
        X = torch.randn((203, 1000), dtype=dt, device="cuda")
        out = torch.empty(1000, dtype=torch.float64, device="cuda")
        _lib.call("bmm_norms", _lib.matrix_dtype(X), X.data_ptr(), 203, 1000, 1000, 0, None, 0, 0, 0, 1, 0,
                  out.data_ptr(), None, _lib.stream_ptr())
        ref = (X.double() ** 2).sum(0)
        assert torch.allclose(out, ref, rtol=1e-12), dt


for name, fn in (("f32", f32), ("f64", f64), ("wide", wide)):
    if part in ("all", name):
        fn()
        torch.cuda.synchronize()
        print(f"{name}: ok", flush=True)
