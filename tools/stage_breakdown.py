"""Per-stage device time of the pipeline in a real (warm) step: events after
every C-ABI call.  Usage: python tools/stage_breakdown.py [cfg2|cfg5|cfg4]"""
import collections
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import workloads  # noqa: E402
from paper_2105_04940_b200.pipeline import SketchPipeline, seeds_from_keys, seeds_from_rngs  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
torch.cuda.set_device(0)
agg = collections.OrderedDict()
if which == "cfg2":
    M, N, sizes = workloads.cfg2()
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    runs = [(cb, W, m) for cb, W in zip((10, 20, 40), (4000, 8000, 16000)) for m in ("OPL", "ONC", "ONMCNR")]
    pipes = [SketchPipeline(500, 20000, 500, sizes, W, m, c0=500) for _, W, m in runs]
    for rep in range(3):
        total = 0.0
        for (cb, W, meth), pipe in zip(runs, pipes):
            st = pipe.stage_times(Md, Nd, seeds_from_rngs(meth, [workloads.sample_rng(2, cb)], len(sizes)))
            for name, ms in st:
                if rep == 2:
                    agg[f"{meth:7s} {name}"] = agg.get(f"{meth:7s} {name}", 0.0) + ms
                total += ms
        print(f"rep {rep}: step {total:.3f} ms")
else:
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import bench
    Md, Nd, sizes, B = bench.device_data(torch, which)
    m, n = Md.shape[-2:]
    p = Nd.shape[-1]
    W = 1024 if which == "cfg5" else 32768
    pipe = SketchPipeline(m, n, p, sizes, W, "ONC", batch=B, dtype=torch.float32)
    seeds = seeds_from_keys("ONC", workloads.ROOT, (int(which[-1]), 1), np.arange(B), len(sizes))
    for rep in range(3):
        st = pipe.stage_times(Md, Nd, seeds)
        print(f"rep {rep}: step {sum(ms for _, ms in st):.3f} ms")
    for name, ms in st:
        agg[name] = agg.get(name, 0.0) + ms
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{v:9.3f} ms  {k}")
