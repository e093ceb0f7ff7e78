"""Time the K1 kernels alone (colsq of M, rowsq of N) on the config shapes:
achieved GB/s and fraction of the measured HBM peak.  Usage: python tools/norms_sweep.py"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_04940_b200 import _lib  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6650.0) \
    if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
torch.cuda.set_device(0)
lib, st = _lib.load(), _lib.stream_ptr()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
# BMM_FLUSH=wr: after the 256 MB write, read a second 256 MB buffer so the L2 holds
# clean lines and the kernel is not charged the write-back of the flush itself
flush_rd = torch.ones(64 << 20, dtype=torch.float32, device="cuda") \
    if __import__("os").environ.get("BMM_FLUSH") == "wr" else None
# rowsq shapes (N: rows x p) and colsq shapes (M: m x n) of the configs
ROWS = [("cfg2 N 20000x500 f64", torch.float64, 1, 20000, 500), ("cfg3 N 100000x1000 f64", torch.float64, 1, 100000, 1000),
        ("cfg5 N 1024x(4096x256) f32", torch.float32, 1024, 4096, 256),
        ("cfg4 N 65536x16384 f32 (1/4)", torch.float32, 1, 65536, 16384)]
COLS = [("cfg2 M 500x20000 f64", torch.float64, 1, 500, 20000), ("cfg3 M 1000x100000 f64", torch.float64, 1, 1000, 100000),
        ("cfg5 M 1024x(256x4096) f32", torch.float32, 1024, 256, 4096),
        ("cfg4 M 16384x65536 f32 (1/4)", torch.float32, 1, 16384, 65536)]


def timed(fn, reps=5):
    out = []
    for _ in range(reps):
        flush.fill_(1)
        if flush_rd is not None:
            flush_rd.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return sorted(out)[len(out) // 2]


for kind, shapes in (("rowsq", ROWS), ("colsq", COLS)):
    for name, dt, B, r, c in shapes:
        X = torch.randn((B, r, c), dtype=dt, device="cuda")
        d = _lib.matrix_dtype(X)
        outv = torch.empty(B * max(r, c), dtype=torch.float64, device="cuda")
        nbytes = X.numel() * X.element_size()
        if kind == "rowsq":
            fn = lambda: lib.bmm_norms(d, None, 0, r, 0, 0, X.data_ptr(), c, c, r * c, B, 0, None,  # noqa: E731
                                       outv.data_ptr(), st)
        else:
            fn = lambda: lib.bmm_norms(d, X.data_ptr(), r, c, c, r * c, None, 0, 0, 0, B, 0,  # noqa: E731
                                       outv.data_ptr(), None, st)
        ms = timed(fn)
        print(f"{kind} {name:32s} {ms*1e3:9.1f} us {nbytes/ms/1e6:7.0f} GB/s ({nbytes/ms/1e6/peak:5.1%})", flush=True)
        del X
