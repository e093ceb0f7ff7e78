"""The config-4 column and row sums right after three sampled contractions (the GPU
power-capped, as inside the bench step) and on a rested GPU: per-kernel ms.  For the A/B
switches read at library load (BMM_COLSQ_WIDE_CFG, BMM_COLSQ_WIDE).
  BMM_COLSQ_WIDE_CFG=2 python tools/cfg4_norms_hot_probe.py"""
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2105_04940_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
m, n, p, K = 16384, 262144, 16384, 4096
sizes = (n // K,) * K
Md, Nd = bench.cfg4_shard(torch, (0, m), (0, p))
group = bench.cfg4_group(torch, m, n, p, sizes)
group.run(Md, Nd, bench.cfg4_seeds(K))
group.check()
torch.cuda.synchronize()
lib, st = _lib.load(), _lib.stream_ptr()
P = lambda t: t.data_ptr()  # noqa: E731
sh, q = group.shared, group.pipes[1]
q.split_gather(Md, Nd, st)


def norms():
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    lib.bmm_norms(1, P(Md), m, n, n, 0, None, 0, 0, 0, 1, 0, P(sh.colsq), None, st)
    e[1].record()
    lib.bmm_norms(1, None, 0, n, 0, 0, P(Nd), p, p, 0, 1, 0, None, P(sh.rowsq), st)
    e[2].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])


ref_c, ref_r = sh.colsq.clone(), sh.rowsq.clone()
time.sleep(2.0)
cool = [norms() for _ in range(3)]
hot = []
for _ in range(3):
    for _ in range(3):
        q.split_gemm(st)
    hot.append(norms())
assert os.environ.get('BMM_PROBE_NOCHECK') or (torch.equal(sh.colsq, ref_c) and torch.equal(sh.rowsq, ref_r))
tag = f"WIDE={os.environ.get('BMM_COLSQ_WIDE', '1')} CFG={os.environ.get('BMM_COLSQ_WIDE_CFG', '0')}"
print(f"{tag}: rested colsq {min(c for c, _ in cool):.2f} rowsq {min(r for _, r in cool):.2f} ms | "
      f"after 3 contractions colsq {' '.join(f'{c:.2f}' for c, _ in hot)}  rowsq {' '.join(f'{r:.2f}' for _, r in hot)} ms",
      flush=True)
