"""Race regression: the config-2 sweep's PipelineGroup graph (nine concurrent
branches, shared statistics with g_k forked beside the norm pass, joint
contractions) replayed many times must give bit-identical products, budgets,
draws and norms every time.  This caught a shared-memory race between the
norm pass and the int8 g_k chain (round 2)."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
from paper_2105_04940_b200.pipeline import PipelineGroup, SketchPipeline, seeds_from_rngs  # noqa: E402


def test_group_replays_are_bit_identical():
    cfg = 2
    M_h, N_h, sizes = workloads.cfg2()
    m, n = M_h.shape
    p = N_h.shape[1]
    K = len(sizes)
    runs = [(cb, W, meth) for cb, W in zip((10, 20, 40), (4000, 8000, 16000)) for meth in ("OPL", "ONC", "ONMCNR")]
    Md, Nd = torch.as_tensor(M_h, device="cuda"), torch.as_tensor(N_h, device="cuda")
    seeds = lambda: [seeds_from_rngs(meth, [workloads.sample_rng(cfg, cb)], K) for cb, W, meth in runs]  # noqa: E731
    g = PipelineGroup([SketchPipeline(m, n, p, sizes, W, meth, c0=500) for _, W, meth in runs])
    ref = [o.cpu().clone() for o in g.run(Md, Nd, seeds())]
    ref_cs = g.shared.colsq.cpu().clone()
    ref_cols = [q.columns_host().copy() for q in g.pipes]
    g.capture(Md, Nd)
    bad = []
    for r in range(60):
        out = [o.cpu() for o in g.run(Md, Nd, seeds())]
        if not torch.equal(g.shared.colsq.cpu(), ref_cs):
            bad.append((r, "colsq"))
        for i, (a, b) in enumerate(zip(ref, out)):
            if not torch.equal(a, b) or not np.array_equal(ref_cols[i], g.pipes[i].columns_host()):
                bad.append((r, i))
    assert not bad, bad[:10]
