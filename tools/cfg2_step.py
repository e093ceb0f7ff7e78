"""One warm cfg2 sweep step through the captured pipelines (for ncu launch lists)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import workloads  # noqa: E402
from paper_2105_04940_b200.pipeline import SketchPipeline, seeds_from_rngs  # noqa: E402

torch.cuda.set_device(0)
M, N, sizes = workloads.cfg2()
Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
runs = [(cb, W, m) for cb, W in zip((10, 20, 40), (4000, 8000, 16000)) for m in ("OPL", "ONC", "ONMCNR")]
pipes = [SketchPipeline(500, 20000, 500, sizes, W, m, c0=500) for _, W, m in runs]
for (cb, W, m), p in zip(runs, pipes):
    p.run(Md, Nd, seeds_from_rngs(m, [workloads.sample_rng(2, cb)], len(sizes)))
    p.capture(Md, Nd)
for it in range(2):
    for (cb, W, m), p in zip(runs, pipes):
        p.run(Md, Nd, seeds_from_rngs(m, [workloads.sample_rng(2, cb)], len(sizes)))
torch.cuda.synchronize()
print("cfg2 step ok")
