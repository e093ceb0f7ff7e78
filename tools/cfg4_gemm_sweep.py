"""The config-4 sampled contraction alone (ONC member, fp16 split on CTA pairs): 6 launches
back to back, per-launch ms -- for A/B switches read at library load (BMM_F16_GROUP_M,
BMM_F16_CHUNK).   BMM_F16_GROUP_M=16 python tools/cfg4_gemm_sweep.py"""
import os
import sys
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
st = _lib.stream_ptr()
q = group.pipes[1]
q.split_gather(Md, Nd, st)
for _ in range(2):
    q.split_gemm(st)
torch.cuda.synchronize()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
evs[0].record()
for i in range(6):
    q.split_gemm(st)
    evs[i + 1].record()
torch.cuda.synchronize()
ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(6)]
print(f"GROUP_M={os.environ.get('BMM_F16_GROUP_M', '4')} CHUNK={os.environ.get('BMM_F16_CHUNK', '4')}: "
      f"{' '.join(f'{x:.2f}' for x in ms)} ms", flush=True)
