"""The config-2 sweep's joint contraction (one batched DMMA GEMM per sketch width)
run once between cudaProfilerStart/Stop, for an ncu capture of exactly those
launches:  ncu --profile-from-start off --set full python tools/joint_gemm_probe.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import workloads  # noqa: E402
from paper_2105_04940_b200.pipeline import PipelineGroup, SketchPipeline, seeds_from_rngs  # noqa: E402

torch.cuda.set_device(0)
M, N, sizes = workloads.cfg2()
Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
runs = [(cb, W, m) for cb, W in zip((10, 20, 40), (4000, 8000, 16000)) for m in ("OPL", "ONC", "ONMCNR")]
group = PipelineGroup([SketchPipeline(500, 20000, 500, sizes, W, m, c0=500) for _, W, m in runs])
group.run(Md, Nd, [seeds_from_rngs(m, [workloads.sample_rng(2, cb)], len(sizes)) for cb, W, m in runs])
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush.fill_(1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
group._joint_gemm()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("joint gemm k:", [jg["k"].tolist() for jg in group._jgroups])
