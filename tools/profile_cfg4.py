"""The config-4 hot kernels once each, for ncu (run with --profile-from-start off):
the data generation and one untimed group step happen outside the profiled
range; inside it: the shared norm pass (bmm_norms: colsq_wide + rowsq_tma),
the Gram g_k^2 (segsq_gram), and for the ONC member the split gather and the
tcgen05 contraction.  Usage: ncu --profile-from-start off ... python tools/profile_cfg4.py"""
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
lib, st = _lib.load(), _lib.stream_ptr()
P = lambda t: t.data_ptr()  # noqa: E731
sh, q = group.shared, group.pipes[1]
W = q.W
torch.cuda.cudart().cudaProfilerStart()
lib.bmm_norms(1, P(Md), m, n, n, 0, P(Nd), p, p, 0, 1, 0, P(sh.colsq), P(sh.rowsq), st)
lib.bmm_segsq_gram(1, P(Md), n, 0, P(Nd), p, 0, m, p, P(sh.offsets), K, 0, 1, P(sh.gsq), st)
q.split_gather(Md, Nd, st)   # fp16 split (balance + gather) for these sizes
q.split_gemm(st)              # gemm_f16split_2sm_kernel
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("profiled kernels done")
