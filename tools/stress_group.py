"""Race hunt: replay the cfg2 sweep's PipelineGroup graph (resident) and the
streamed end-to-end graph many times and compare every replay with the first
(bit-identical expected).  Usage: python tools/stress_group.py [reps]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import workloads  # noqa: E402
from paper_2105_04940_b200.pipeline import PipelineGroup, SketchPipeline, seeds_from_rngs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
torch.cuda.set_device(0)
cfg = 2
M_h, N_h, sizes = workloads.cfg2()
m, n = M_h.shape
p = N_h.shape[1]
K = len(sizes)
runs = [(cb, W, meth, 500) for cb, W in zip((10, 20, 40), (4000, 8000, 16000)) for meth in ("OPL", "ONC", "ONMCNR")]
Md, Nd = torch.as_tensor(M_h, device="cuda"), torch.as_tensor(N_h, device="cuda")
seeds = lambda: [seeds_from_rngs(meth, [workloads.sample_rng(cfg, cb)], K) for cb, W, meth, c0 in runs]  # noqa: E731
g = PipelineGroup([SketchPipeline(m, n, p, sizes, W, meth, c0=c0) for _, W, meth, c0 in runs])
ref = [o.cpu().clone() for o in g.run(Md, Nd, seeds())]
refb = [q.budgets_host().copy() for q in g.pipes]
refc = [q.columns_host().copy() for q in g.pipes]
refs = [q.scales_host().copy() for q in g.pipes]
refn = [(q.colsq.cpu().clone(), q.rowsq.cpu().clone(), q.probs.cpu().clone(), q.cum.cpu().clone()) for q in g.pipes]
refk = [q.k_column.cpu().clone() for q in g.pipes]
refst = [q.states.cpu().clone() for q in g.pipes]
g.capture(Md, Nd)
bad = 0
for r in range(reps):
    out = [o.cpu() for o in g.run(Md, Nd, seeds())]
    for i, (a, b) in enumerate(zip(ref, out)):
        if not torch.equal(a, b):
            bad += 1
            q = g.pipes[i]
            same_b = np.array_equal(refb[i], q.budgets_host())
            same_c = np.array_equal(refc[i], q.columns_host())
            same_s = np.array_equal(refs[i], q.scales_host())
            nn = [torch.equal(x, y.cpu()) for x, y in zip(refn[i], (q.colsq, q.rowsq, q.probs, q.cum))]
            same_k = torch.equal(refk[i], q.k_column.cpu())
            same_st = torch.equal(refst[i], q.states.cpu())
            if not nn[0]:
                d = (refn[i][0] - q.colsq.cpu()).abs()
                bad_idx = torch.nonzero(d).flatten()
                rel = (d / refn[i][0].abs().clamp_min(1e-300))[bad_idx]
                print(f"   colsq differs at {bad_idx.numel()} of {d.numel()} columns: first {bad_idx[:8].tolist()} "
                      f"last {bad_idx[-4:].tolist()} rel max {float(rel.max()):.3e} min {float(rel.min()):.3e}",
                      flush=True)
            print(f"resident replay {r} product {i} ({runs[i][2]} W={runs[i][1]}): rel "
                  f"{float((a - b).norm() / a.norm()):.3e} budgets {same_b} cols {same_c} scales {same_s} "
                  f"norms/probs/cum {nn} kcol {same_k} states {same_st}", flush=True)
print(f"resident: {bad} mismatches in {reps} replays", flush=True)
hg = PipelineGroup([SketchPipeline(m, n, p, sizes, W, meth, c0=c0) for _, W, meth, c0 in runs], joint=False)
M_pin, N_pin = torch.from_numpy(M_h).pin_memory(), torch.from_numpy(N_h).pin_memory()
Mx, Nx = torch.empty_like(Md), torch.empty_like(Nd)
outs = [torch.empty((m, p), dtype=torch.float64).pin_memory() for _ in runs]
hg.capture_host(Mx, Nx, M_pin, N_pin, outs, seeds(), n_chunks=8)
bad = 0
first = None
for r in range(reps):
    hg.run_host(seeds())
    torch.cuda.synchronize()
    cur = [o.clone() for o in outs]
    if first is None:
        first = cur
        err = max(float((a - b).norm() / a.norm()) for a, b in zip(ref, cur))
        print(f"host vs resident (first): max rel {err:.3e}", flush=True)
        continue
    for i, (a, b) in enumerate(zip(first, cur)):
        if not torch.equal(a, b):
            bad += 1
            print(f"host replay {r} product {i}: rel {float((a - b).norm() / a.norm()):.3e}", flush=True)
print(f"host: {bad} mismatches in {reps} replays", flush=True)
