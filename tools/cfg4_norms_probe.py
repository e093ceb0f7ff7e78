"""Config-4 norm pass at full size: colsq(M 16384x262144 f32), rowsq(N 262144x16384
f32) alone, back to back (bmm_norms) and on two concurrent streams; GB/s and the
fraction of MEASURED_PEAKS hbm_gbs.  A/B variants through the BMM_* env switches
of csrc/norms.cu (one process per variant).  Usage: python tools/cfg4_norms_probe.py"""
import json
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2105_04940_b200 import _lib  # noqa: E402

peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6538.6) \
    if (ROOT / "MEASURED_PEAKS.json").exists() else 6538.6
torch.cuda.set_device(0)
lib, st = _lib.load(), _lib.stream_ptr()
m, n, p = 16384, 262144, 16384
M = torch.randn((m, n), dtype=torch.float32, device="cuda")
N = torch.randn((n, p), dtype=torch.float32, device="cuda")
cs = torch.empty(n, dtype=torch.float64, device="cuda")
rs = torch.empty(n, dtype=torch.float64, device="cuda")
s2 = torch.cuda.Stream()


def timed(fn, reps=5):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return sorted(out)[len(out) // 2]


def both_concurrent():
    cur = torch.cuda.current_stream()
    s2.wait_stream(cur)
    lib.bmm_norms(1, M.data_ptr(), m, n, n, 0, None, p, p, 0, 1, 0, cs.data_ptr(), None, st)
    with torch.cuda.stream(s2):
        lib.bmm_norms(1, None, m, n, n, 0, N.data_ptr(), p, p, 0, 1, 0, None, rs.data_ptr(), s2.cuda_stream)
    cur.wait_stream(s2)


half = 4.0 * m * n
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("BMM_")) or "default"
for name, fn, nb in [(k, f, b) for k, f, b in (
        ("colsq M", lambda: lib.bmm_norms(1, M.data_ptr(), m, n, n, 0, None, p, p, 0, 1, 0, cs.data_ptr(), None, st), half),
        ("rowsq N", lambda: lib.bmm_norms(1, None, m, n, n, 0, N.data_ptr(), p, p, 0, 1, 0, None, rs.data_ptr(), st), half),
        ("bmm_norms M+N", lambda: lib.bmm_norms(1, M.data_ptr(), m, n, n, 0, N.data_ptr(), p, p, 0, 1, 0, cs.data_ptr(),
                                                rs.data_ptr(), st), 2 * half),
        ("two streams M||N", both_concurrent, 2 * half)) if os.environ.get("BMM_PROBE_ONLY", k) in k]:
    ms = timed(fn)
    print(f"[{tag}] {name:18s} {ms:8.3f} ms {nb / ms / 1e6:7.0f} GB/s ({nb / ms / 1e6 / peak:5.1%})", flush=True)
