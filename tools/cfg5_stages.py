"""Per-stage device times of the config-5 pipeline (eager, an event after every
C-ABI call): where the non-norm, non-contraction time of the step goes.

  python tools/cfg5_stages.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2105_04940_b200.pipeline import SketchPipeline, seeds_from_keys  # noqa: E402


def main():
    torch.cuda.set_device(0)
    Md, Nd, sizes, B = bench.device_data(torch, "cfg5")
    m, n = Md.shape[-2:]
    p = Nd.shape[-1]
    K = len(sizes)
    pipe = SketchPipeline(m, n, p, sizes, 1024, "ONC", batch=B, dtype=torch.float32)
    seeds = seeds_from_keys("ONC", workloads.ROOT, (5, 1), np.arange(B), K)
    pipe.run(Md, Nd, seeds)
    torch.cuda.synchronize()
    acc = {}
    for _ in range(5):
        for name, ms in pipe.stage_times(Md, Nd, seeds):
            acc.setdefault(name, []).append(ms)
    tot = 0.0
    for name, v in acc.items():
        med = float(np.median(v))
        tot += med
        print(f"{name:34s} {med:8.3f} ms")
    print(f"{'sum':34s} {tot:8.3f} ms")


if __name__ == "__main__":
    main()
