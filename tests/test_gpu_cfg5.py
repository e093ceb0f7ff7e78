"""Config 5 at full size: all 4096 problems (float32 256x4096 . 4096x256, K=64
blocks of 64, per-problem seeds) as the bench generates and runs them.
* ONC with W=1024: every problem's norms bit-exact (oracle on the float64
  upcast), its probabilities, budgets, draws and scales bit-exact, C.D of a
  problem subset within 1e-5 of float64 of the same sketch;
* OPL (Gram g_k^2) and SSM (16 draws) cells: budgets / draws of every problem
  bit-exact to the oracle's plan from the device statistics, g_k^2 of a subset
  of problems against the oracle's multiplied-out blocks (1e-12)."""
import numpy as np
import pytest

import workloads
from oracle import blockmm_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")


def _draws(probs, sizes, budgets, streams):
    off = O.offsets_of(sizes)
    cols, scales = [], []
    for k in range(len(sizes)):
        if budgets[k]:
            pk = probs[off[k]:off[k + 1]]
            idx = O.draw(pk, int(budgets[k]), streams[k])
            cols.append(off[k] + idx)
            scales.append(1.0 / np.sqrt(int(budgets[k]) * pk[idx]))
    return np.concatenate(cols), np.concatenate(scales)


def test_cfg5_all_problems():
    import bench
    from paper_2105_04940_b200.pipeline import SketchPipeline, seeds_from_keys, seeds_from_rngs

    Md, Nd, sizes, B = bench.device_data(torch, "cfg5")
    m, n, p, K, W = 256, 4096, 256, 64, 1024
    keys = np.arange(B)
    onc = SketchPipeline(m, n, p, sizes, W, "ONC", batch=B, dtype=torch.float32)
    CD = onc.run(Md, Nd, seeds_from_keys("ONC", workloads.ROOT, (5, 1), keys, K))
    onc.check()
    opl = SketchPipeline(m, n, p, sizes, W, "OPL", batch=B, dtype=torch.float32)
    assert opl.seg_engine == "gram"
    opl.run(Md, Nd, seeds_from_keys("OPL", workloads.ROOT, (5, 2), keys, K))
    opl.check()
    ssm = SketchPipeline(m, n, p, sizes, 0, "SSM", batch=B, draws=16, dtype=torch.float32)
    ssm.run(Md, Nd, seeds_from_rngs("SSM", [workloads.sample_rng(5, 3, int(b)) for b in keys], K, draws=16))
    ssm.check()

    cs_all = onc.colsq.view(B, n).cpu().numpy()
    rs_all = onc.rowsq.view(B, n).cpu().numpy()
    bud_onc, col_onc, sc_onc = onc.budgets_host(), onc.columns_host(), onc.scales_host()
    bud_opl, col_opl, sc_opl = opl.budgets_host(), opl.columns_host(), opl.scales_host()
    gsq_all = opl.gsq.view(B, K).cpu().numpy()
    blk_ssm, sc_ssm = ssm.columns_host(), ssm.scales_host()
    off = O.offsets_of(sizes)
    for b0 in range(0, B, 256):
        Mh = Md[b0:b0 + 256].cpu().numpy()
        Nh = Nd[b0:b0 + 256].cpu().numpy()
        for j in range(Mh.shape[0]):
            b = b0 + j
            M64, N64 = Mh[j].astype(np.float64), Nh[j].astype(np.float64)
            cs, rs = O.colsq(M64), O.rowsq(N64)
            assert np.array_equal(cs_all[b], cs) and np.array_equal(rs_all[b], rs), b
            probs, s = O.block_stats(cs, rs, sizes)
            bud, _ = O.plan_budgets("ONC", sizes, W, s=s)
            cols, scales = _draws(probs, sizes, bud, workloads.sample_rng(5, b).spawn(K))
            assert np.array_equal(bud_onc[b], bud) and np.array_equal(col_onc[b], cols), b
            assert np.array_equal(sc_onc[b], scales), b
            bud, _ = O.plan_budgets("OPL", sizes, W, s=s, aux_sq=gsq_all[b])
            rng = np.random.default_rng(np.random.SeedSequence(workloads.ROOT, spawn_key=(5, 2, b)))
            cols, scales = _draws(probs, sizes, bud, rng.spawn(K))
            assert np.array_equal(bud_opl[b], bud) and np.array_equal(col_opl[b], cols), b
            assert np.array_equal(sc_opl[b], scales), b
            q = O.block_norm_weights(cs, rs, sizes)
            q = q / q.sum()
            blocks = O.draw(q, 16, workloads.sample_rng(5, 3, b))
            assert np.array_equal(blk_ssm[b], blocks), b
            np.testing.assert_allclose(sc_ssm[b], 1.0 / np.sqrt(16 * q[blocks]), rtol=1e-13)
            if b % 512 == 0:  # g_k^2 and C.D on a subset
                gsq = O.block_product_sq(M64, N64, sizes)
                np.testing.assert_allclose(gsq_all[b], gsq, rtol=1e-12)
                C64 = M64[:, col_onc[b]] * sc_onc[b]
                D64 = N64[col_onc[b], :] * sc_onc[b][:, None]
                ref = C64 @ D64
                got = CD[b].double().cpu().numpy()
                assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-5, b
