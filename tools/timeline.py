"""Where a PipelineGroup step spends its time inside ONE graph replay: every
pipeline of the group records a device clock stamp (bmm_timestamp, %globaltimer)
after each of its C-ABI calls, the group graph is captured with the stamps and
replayed; prints per branch the end time of every stage relative to the step start.
Usage: python tools/timeline.py [reps] [cfg2|cfg4]   (cfg2: the nine-product sweep;
cfg4: the default bench step -- shared stats + OPL, ONC, SSM at full size)"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import workloads  # noqa: E402
from paper_2105_04940_b200 import _lib  # noqa: E402
from paper_2105_04940_b200.pipeline import PipelineGroup, SketchPipeline, seeds_from_rngs  # noqa: E402

torch.cuda.set_device(0)
WORKLOAD = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
if WORKLOAD == "cfg4":
    import bench  # noqa: E402
    Md, Nd, sizes, _ = bench.device_data(torch, "cfg4")
    group = bench.cfg4_group(torch, Md.shape[0], Md.shape[1], Nd.shape[1], sizes)
    pipes = group.pipes
    runs = [(rep, w, meth) for meth, w, rep in bench.CFG4_RUNS]
    seeds = lambda: bench.cfg4_seeds(len(sizes))  # noqa: E731
else:
    M, N, sizes = workloads.cfg2()
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    runs = [(cb, W, m) for cb, W in zip((10, 20, 40), (4000, 8000, 16000)) for m in ("OPL", "ONC", "ONMCNR")]
    pipes = [SketchPipeline(500, 20000, 500, sizes, W, m, c0=500) for _, W, m in runs]
    group = PipelineGroup(pipes)
    seeds = lambda: [seeds_from_rngs(m, [workloads.sample_rng(2, cb)], len(sizes)) for cb, W, m in runs]  # noqa: E731
group.run(Md, Nd, seeds())
start = torch.zeros(1, dtype=torch.int64, device="cuda")
end = torch.zeros(1, dtype=torch.int64, device="cuda")
sh = group.shared  # the shared statistics stage (norms, probabilities, g_k once per step)
for p in pipes + ([sh] if sh is not None else []):
    p.stamps = (torch.zeros(256, dtype=torch.int64, device="cuda"), [])
lib = _lib.load()
# capture: a stamp at the start (before the fork) and one after the join
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    group._launch_all(Md, Nd)
torch.cuda.current_stream().wait_stream(side)
for p in pipes + ([sh] if sh is not None else []):
    p.stamps[1].clear()
streams = group._branch_streams()
group._active(True)
with torch.cuda.graph(g):
    cap = torch.cuda.current_stream()
    lib.bmm_timestamp(start.data_ptr(), _lib.stream_ptr())
    evs = None
    if sh is not None:
        *evs, ss = group._fork_stats(cap, Md, Nd)
        streams.append(ss)
    for s, p in zip(streams, pipes):
        s.wait_stream(cap)
        group._member_wait(s, p, evs)
        with torch.cuda.stream(s):
            p.launch(Md, Nd)
    for jg in group._jgroups:
        js = torch.cuda.Stream()
        for i in jg["idx"]:
            js.wait_stream(streams[i])
        with torch.cuda.stream(js):
            group._joint_gemm(jg)
            lib.bmm_timestamp(end.data_ptr() + 0, _lib.stream_ptr())  # overwritten: last one wins
        streams.append(js)
    for s in streams:
        cap.wait_stream(s)
    lib.bmm_timestamp(end.data_ptr(), _lib.stream_ptr())
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
rows = []
for r in range(reps):
    for p, sd in zip(pipes, seeds()):
        p.set_seeds(sd)
    g.replay()
    torch.cuda.synchronize()
    t0 = int(start.item())
    rows.append((t0, int(end.item()), [(p.stamps[1], p.stamps[0][:len(p.stamps[1])].cpu().numpy() - t0) for p in pipes]))
group._active(False)
t0, t1, br = rows[-1]
if sh is not None:
    names, ts = sh.stamps[1], sh.stamps[0][:len(sh.stamps[1])].cpu().numpy() - t0
    print("shared  stats   done at " + f"{ts[-1] / 1e3:7.1f} us | " +
          " ".join(f"{nm.replace('bmm_', '')}:{t / 1e3:.0f}" for nm, t in zip(names, ts)))
print(f"step (stamp to stamp): {(t1 - t0) / 1e3:.1f} us  (reps: {[round((b - a) / 1e3, 1) for a, b, _ in rows]})")
for (cb, W, meth), (names, ts) in zip(runs, br):
    prev = 0
    parts = []
    for nm, t in zip(names, ts):
        parts.append(f"{nm.replace('bmm_', '')}:{t / 1e3:.0f}")
        prev = t
    print(f"{meth:7s} W={W:5d} done at {prev / 1e3:7.1f} us | " + " ".join(parts))
