"""One pass of each hot kernel at profiling-friendly sizes, for ncu captures.

cfg5-shaped float32 batch (512 problems, ONC, W=1024): norms, plan, sampler,
split gather, tcgen05 3xTF32 GEMM; cfg2-shaped float64 ONC at W=16000:
norms, plan, sampler, gather, DMMA GEMM; cfg2 OPL: segmented square sums
(int8 Ozaki path); cfg3-shaped float64 contraction on the int8 Ozaki path.
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import workloads  # noqa: E402
from paper_2105_04940_b200.pipeline import SketchPipeline, seeds_from_keys, seeds_from_rngs  # noqa: E402

torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(5)
B, m, n, p, K, W = 512, 256, 4096, 256, 64, 1024
M = torch.randn((B, m, n), generator=g, device="cuda") * torch.randn((B, 1, n), generator=g, device="cuda").exp()
N = torch.randn((B, n, p), generator=g, device="cuda") * torch.randn((B, n, 1), generator=g, device="cuda").exp()
pipe = SketchPipeline(m, n, p, (64,) * K, W, "ONC", batch=B, dtype=torch.float32)
pipe.run(M, N, seeds_from_keys("ONC", workloads.ROOT, (5, 1), np.arange(B), K))
pipe.check()

M2, N2, sizes = workloads.cfg2()
Md, Nd = torch.as_tensor(M2, device="cuda"), torch.as_tensor(N2, device="cuda")
pipe2 = SketchPipeline(500, 20000, 500, sizes, 16000, "ONC")
pipe2.run(Md, Nd, seeds_from_rngs("ONC", [workloads.sample_rng(2, 40)], len(sizes)))
pipe2.check()
pipe3 = SketchPipeline(500, 20000, 500, sizes, 16000, "OPL")  # + segmented square sums (g_k)
pipe3.run(Md, Nd, seeds_from_rngs("OPL", [workloads.sample_rng(2, 40)], len(sizes)))
pipe3.check()
# cfg3-shaped float64 sampled contraction on the int8 Ozaki path (1000 x 17000 x 1000)
from paper_2105_04940_b200 import _lib  # noqa: E402
A3 = torch.randn((1000, 17000), generator=g, device="cuda", dtype=torch.float64)
B3 = torch.randn((17000, 1000), generator=g, device="cuda", dtype=torch.float64)
O3 = torch.empty((1000, 1000), dtype=torch.float64, device="cuda")
ws3 = _lib.workspace(_lib.load().bmm_gemm_i8_workspace(1000, 1000, 17000, 1))
_lib.call("bmm_gemm_i8", 0, A3.data_ptr(), 17000, 0, B3.data_ptr(), 1000, 0, 1000, 1000, 17000, None, None, 1,
          O3.data_ptr(), 1000, 0, ws3.data_ptr(), ws3.numel(), _lib.stream_ptr())
torch.cuda.synchronize()
print("profile_kernels ok")
