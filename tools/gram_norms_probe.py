"""Config-4 statistics stage, kernel by kernel (cool GPU, CUDA events):
the norm pass alone, the Gram-form g_k^2 alone, and the Gram kernel with the
norm pass fused in (BMM_GRAM_NORMS_SIDES=3: colsq and rowsq; =1: colsq only,
then the rowsq-only norm kernel).

  BMM_GRAM_NORMS_SIDES=3 python tools/gram_norms_probe.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2105_04940_b200 import _lib  # noqa: E402


def timed(fn, reps=3):
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out))


def main():
    torch.cuda.set_device(0)
    Md, Nd, sizes, _ = bench.device_data(torch, "cfg4")
    m, n = Md.shape
    p = Nd.shape[1]
    K = len(sizes)
    off = torch.as_tensor(np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64), device="cuda")
    gsq = torch.empty(K, dtype=torch.float64, device="cuda")
    cs = torch.empty(n, dtype=torch.float64, device="cuda")
    rs = torch.empty(n, dtype=torch.float64, device="cuda")
    cs2, rs2 = torch.empty_like(cs), torch.empty_like(rs)
    st = _lib.stream_ptr()
    P = lambda t: t.data_ptr()  # noqa: E731
    lib = _lib.load()
    norms = lambda: lib.bmm_norms(1, P(Md), m, n, n, 0, P(Nd), p, p, 0, 1, 0, P(cs), P(rs), st)  # noqa: E731
    rows_only = lambda: lib.bmm_norms(1, None, 0, n, 0, 0, P(Nd), p, p, 0, 1, 0, None, P(rs2), st)  # noqa: E731
    gram = lambda: lib.bmm_segsq_gram(1, P(Md), n, 0, P(Nd), p, 0, m, p, P(off), K, 0, 1, P(gsq), st)  # noqa: E731
    fused = lambda: lib.bmm_segsq_gram_norms(1, P(Md), n, 0, P(Nd), p, 0, m, p, P(off), K, 0, 1, P(gsq),  # noqa
                                             P(cs2), P(rs2), n, st)
    sides = os.environ.get("BMM_GRAM_NORMS_SIDES", "3")
    for f in (norms, gram, fused, rows_only):
        f()
    torch.cuda.synchronize()
    t_n, t_g, t_f = timed(norms), timed(gram), timed(fused)
    line = f"sides={sides}: norms {t_n:.2f} ms, gram {t_g:.2f} ms, gram+norms fused {t_f:.2f} ms"
    if sides == "1":
        t_r = timed(rows_only)
        line += f" + rowsq alone {t_r:.2f} ms"
    fused()
    rows_only() if sides == "1" else None
    torch.cuda.synchronize()
    line += f"; colsq equal {torch.equal(cs, cs2)}, rowsq equal {torch.equal(rs, rs2)}"
    print(line, flush=True)


if __name__ == "__main__":
    main()
