"""Time bmm_block_probs on the cfg2 instance: full (probs, s, CDF) and without the CDF."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import workloads  # noqa: E402
from paper_2105_04940_b200 import _lib  # noqa: E402

M, N, sizes = workloads.cfg2()
n = M.shape[1]
K = len(sizes)
colsq = torch.as_tensor((M * M).sum(0), device="cuda")
rowsq = torch.as_tensor((N * N).sum(1), device="cuda")
off = _lib.i64(np.concatenate([[0], np.cumsum(sizes)]))
probs = torch.empty(n, dtype=torch.float64, device="cuda")
cum = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.empty(K, dtype=torch.float64, device="cuda")
last = torch.empty(K, dtype=torch.int64, device="cuda")
st = _lib.stream_ptr()
P = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
print("max block", max(sizes))
for name, c, l, ss in (("full", cum, last, s), ("no cdf", None, None, s), ("no cdf, no s", None, None, None)):
    for _ in range(3):
        _lib.call("bmm_block_probs", P(colsq), P(rowsq), n, P(off), K, 1, max(sizes), P(probs), P(ss), None, P(c), P(l), st)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        _lib.call("bmm_block_probs", P(colsq), P(rowsq), n, P(off), K, 1, max(sizes), P(probs), P(ss), None, P(c), P(l), st)
    b.record()
    torch.cuda.synchronize()
    print(name, a.elapsed_time(b) / 20 * 1e3, "us")
