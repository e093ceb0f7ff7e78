"""Host <-> device transfers of the drop-in API from pageable memory: plain .cpu() / .to(device)
against the staged copies in _lib (two pinned buffers, threaded memcpy), by size -- picks the
threshold _lib._BIG.

  python tools/host_copy_probe.py [MB ...]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_04940_b200 import _lib  # noqa: E402


def best(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        del r
    return float(np.median(ts))


def main():
    sizes = [float(x) for x in sys.argv[1:]] or [2, 8, 16, 32, 64, 256, 4300]
    _lib.host(torch.zeros(1 << 21, dtype=torch.float64, device="cuda"))  # staging buffers exist
    for mb in sizes:
        n = int(mb * 1e6 / 8)
        t = torch.arange(n, dtype=torch.float64, device="cuda")
        a = np.arange(n, dtype=np.float64)
        row = []
        for big in (1 << 60, 0):  # plain, staged
            _lib._BIG = big
            row.append(best(lambda: _lib.host(t)))
            row.append(best(lambda: _lib.to_device(a)))
        assert np.array_equal(_lib.host(t), a) and torch.equal(_lib.to_device(a), t)
        print(f"{mb:7.0f} MB  D2H plain {row[0] * 1e3:8.2f} ms  staged {row[2] * 1e3:8.2f} ms   "
              f"H2D plain {row[1] * 1e3:8.2f} ms  staged {row[3] * 1e3:8.2f} ms", flush=True)


if __name__ == "__main__":
    main()
