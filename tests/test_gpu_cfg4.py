"""Config 4 at full size (M 16384 x 262144, N 262144 x 16384 float32, K=4096,
W=32768, ONC): norms, budgets, sampled indices and scales bit-exact against the
NumPy oracle (norms restated chunk-by-chunk with the exact sequential
continuation, on the float64 upcast); C.D against a float64 product of the
same sketch on a 256-row slab within 1e-5."""
import numpy as np
import pytest

import workloads
from oracle import blockmm_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")


def test_cfg4_full_size_parity():
    import bench
    from paper_2105_04940_b200.pipeline import SketchPipeline, seeds_from_keys

    Md, Nd, sizes, _ = bench.device_data(torch, "cfg4")
    m, n = Md.shape
    p = Nd.shape[1]
    K, W = len(sizes), 32768
    pipe = SketchPipeline(m, n, p, sizes, W, "ONC", dtype=torch.float32)
    CD = pipe.run(Md, Nd, seeds_from_keys("ONC", workloads.ROOT, (4, 1), [0], K))
    pipe.check()

    # oracle norm pass on host copies (float64 upcast, exact chunk continuation)
    acc = None
    for r0 in range(0, m, 256):
        sl = Md[r0:r0 + 256].cpu().numpy().astype(np.float64)
        sq = sl * sl
        if acc is not None:
            sq = np.concatenate([acc[None, :], sq], axis=0)
        acc = np.add.reduce(sq, axis=0)
    colsq = acc
    rowsq = np.empty(n)
    for r0 in range(0, n, 4096):
        sl = Nd[r0:r0 + 4096].cpu().numpy().astype(np.float64)
        rowsq[r0:r0 + 4096] = np.add.reduce(sl * sl, axis=1)
    assert np.array_equal(pipe.colsq.cpu().numpy(), colsq)
    assert np.array_equal(pipe.rowsq.cpu().numpy(), rowsq)

    probs, s = O.block_stats(colsq, rowsq, sizes)
    budgets, _ = O.plan_budgets("ONC", sizes, W, s=s)
    assert np.array_equal(pipe.budgets_host()[0], budgets)
    streams = workloads.sample_rng(4).spawn(K)
    off = O.offsets_of(sizes)
    cols, scales = [], []
    for k in range(K):
        if budgets[k]:
            pk = probs[off[k]:off[k + 1]]
            idx = O.draw(pk, int(budgets[k]), streams[k])
            cols.append(off[k] + idx)
            scales.append(1.0 / np.sqrt(int(budgets[k]) * pk[idx]))
    cols, scales = np.concatenate(cols), np.concatenate(scales)
    assert np.array_equal(pipe.columns_host()[0], cols)
    assert np.array_equal(pipe.scales_host()[0], scales)

    # C.D on a row slab against float64 of the same sketch
    ci = torch.as_tensor(cols, device="cuda")
    sc = torch.as_tensor(scales, device="cuda")
    C64 = Md[:256].index_select(1, ci).double() * sc
    D64 = Nd.index_select(0, ci).double() * sc[:, None]
    ref = C64 @ D64
    err = ((CD[:256].double() - ref).norm() / ref.norm()).item()
    assert err < 1e-5, err
