"""Time bmm_segsq_gram_gather on pilot shapes: python tools/gram_probe.py m n p K L"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_04940_b200 import _lib  # noqa: E402

m, n, p, K, L = (int(x) for x in sys.argv[1:6])
g = np.random.default_rng(0)
M = torch.as_tensor(g.standard_normal((m, n)), device="cuda")
N = torch.as_tensor(g.standard_normal((n, p)), device="cuda")
W = K * L
col = _lib.i64(np.sort(g.integers(0, n, W)))
sc = torch.as_tensor(g.uniform(0.5, 2, W), device="cuda")
seg = _lib.i64(np.arange(K + 1) * L)
out = torch.empty(K, dtype=torch.float64, device="cuda")
st = _lib.stream_ptr()
f = lambda: _lib.call("bmm_segsq_gram_gather", 0, M.data_ptr(), n, 0, N.data_ptr(), p, 0, m, p, col.data_ptr(),  # noqa
                      sc.data_ptr(), W, seg.data_ptr(), K, 0, L, 1, out.data_ptr(), st)
for _ in range(3):
    f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    f()
b.record()
torch.cuda.synchronize()
print(f"gram m={m} n={n} p={p} K={K} L={L}: {a.elapsed_time(b) / 20 * 1e3:.1f} us")
