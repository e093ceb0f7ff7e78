"""Where a bmm_plan_small CTA spends its time at config 5: SM-clock stamps at the stage
boundaries of every problem (bmm_plan_small_debug), medians over the problems.

  python tools/plan_small_probe.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2105_04940_b200 import _lib  # noqa: E402
from paper_2105_04940_b200.pipeline import SketchPipeline, seeds_from_keys  # noqa: E402

STAGES = ["offsets+scores", "probs+cdf (thread per block)", "probs write", "budgets", "streams", "draws",
          "compress", "balance"]


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
    dbg = torch.zeros((B, 16), dtype=torch.int64, device="cuda")
    _lib.call("bmm_plan_small_debug", dbg.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pipe._plan_small_call(_lib.stream_ptr())
    e1.record()
    torch.cuda.synchronize()
    _lib.call("bmm_plan_small_debug", None)
    t = dbg.cpu().numpy()
    d = np.diff(t[:, :8], axis=1)
    print(f"kernel {e0.elapsed_time(e1) * 1e3:.0f} us for {B} problems")
    names = ["scores+probs+cdf", "cum write", "budgets", "streams", "draws", "compress", "balance"]
    for i in range(7):
        print(f"{names[i]:18s} median {np.median(d[:, i]):9.0f} clk   p90 {np.percentile(d[:, i], 90):9.0f}")
    # inside the first stage, block 0's group: stamps 8..13 after the stage's start (stamp 0)
    fine = ["setup+loads+scores", "two sums", "normalise x2 + sum", "probs write", "other rounds", "cdf chains"]
    prev = t[:, 0]
    for i, nm in zip(range(8, 14), fine):
        print(f"  {nm:18s} median {np.median(t[:, i] - prev):9.0f} clk")
        prev = t[:, i]
    tot = t[:, 7] - t[:, 0]
    print(f"{'CTA total':14s} median {np.median(tot):9.0f} clk   p90 {np.percentile(tot, 90):9.0f}")


if __name__ == "__main__":
    main()
