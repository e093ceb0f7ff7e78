import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import workloads
from paper_2105_04940_b200.pipeline import PipelineGroup, SketchPipeline, seeds_from_rngs
torch.cuda.set_device(0)
cfg = 2
M_h, N_h, sizes = workloads.cfg2()
m, n = M_h.shape; p = N_h.shape[1]; K = len(sizes)
runs = [(cb, W, meth, 500) for cb, W in zip((10, 20, 40), (4000, 8000, 16000)) for meth in ("OPL", "ONC", "ONMCNR")]
Md, Nd = torch.as_tensor(M_h, device="cuda"), torch.as_tensor(N_h, device="cuda")
seeds = lambda: [seeds_from_rngs(meth, [workloads.sample_rng(cfg, cb)], K) for cb, W, meth, c0 in runs]
for joint in (False, True):
    g = PipelineGroup([SketchPipeline(m, n, p, sizes, W, meth, c0=c0) for _, W, meth, c0 in runs], joint=joint)
    eager = [o.cpu().clone() for o in g.run(Md, Nd, seeds())]
    g.capture(Md, Nd)
    rep = [o.cpu().clone() for o in g.run(Md, Nd, seeds())]
    print("joint", joint, "eager vs replay:", [float((a - b).norm() / a.norm()) for a, b in zip(eager, rep)])
    hg = PipelineGroup([SketchPipeline(m, n, p, sizes, W, meth, c0=c0) for _, W, meth, c0 in runs], joint=False)
    M_pin = torch.from_numpy(M_h).pin_memory(); N_pin = torch.from_numpy(N_h).pin_memory()
    Mx, Nx = torch.empty_like(Md), torch.empty_like(Nd)
    outs = [torch.empty((m, p), dtype=torch.float64).pin_memory() for _ in runs]
    hg.capture_host(Mx, Nx, M_pin, N_pin, outs, seeds(), n_chunks=8)
    hg.run_host(seeds()); torch.cuda.synchronize()
    print("joint", joint, "host vs eager:", [float((a - b).norm() / a.norm()) for a, b in zip(eager, outs)])
    print("Mx equal", torch.equal(Mx.cpu(), torch.from_numpy(M_h)), "Nx equal", torch.equal(Nx.cpu(), torch.from_numpy(N_h)))
    print("budgets equal", [np.array_equal(a.budgets_host(), b.budgets_host()) for a, b in zip(g.pipes, hg.pipes)])
    print("cols equal", [np.array_equal(a.columns_host(), b.columns_host()) for a, b in zip(g.pipes, hg.pipes)])
