"""Config 4 at full size (M 16384 x 262144, N 262144 x 16384 float32, K=4096
blocks of 64): the benched step -- OPL and ONC with W=32768 and SSM with 512
draws over one shared statistics stage -- against the NumPy oracle.
* norms: every column of M and every row of N bit-exact, restated chunk by chunk
  with the exact sequential continuation on the float64 upcast (the full upcast
  needs 69 GB);
* plan and draws: probabilities, score sums, ONC/OPL budgets, every draw and
  scale bit-exact; SSM block probabilities (1e-13) and draws (bench.cfg4_parity);
* g_k^2 of sampled blocks vs the oracle's multiplied-out blocks (1e-12);
* C.D on 4 row slabs (first, last, two inner) vs float64 of the same sketch (1e-5)."""
import numpy as np
import pytest

from oracle import blockmm_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")


def test_cfg4_full_size_parity():
    import bench

    m, n, p, K = 16384, 262144, 16384, 4096
    Md, Nd = bench.cfg4_shard(torch, (0, m), (0, p))
    group = bench.cfg4_group(torch, m, n, p, (n // K,) * K)
    outs = [o.clone() for o in group.run(Md, Nd, bench.cfg4_seeds(K))]
    group.check()

    # oracle norm pass on host copies (float64 upcast, exact chunk continuation)
    acc = None
    for r0 in range(0, m, 256):
        sl = Md[r0:r0 + 256].cpu().numpy().astype(np.float64)
        sq = sl * sl
        if acc is not None:
            sq = np.concatenate([acc[None, :], sq], axis=0)
        acc = np.add.reduce(sq, axis=0)
    rowsq = np.empty(n)
    for r0 in range(0, n, 4096):
        sl = Nd[r0:r0 + 4096].cpu().numpy().astype(np.float64)
        rowsq[r0:r0 + 4096] = np.add.reduce(sl * sl, axis=1)
    assert np.array_equal(group.shared.colsq.cpu().numpy(), acc)
    assert np.array_equal(group.shared.rowsq.cpu().numpy(), rowsq)

    res = bench.cfg4_cpu_leg_parity(torch, group, Md, Nd, outs)  # raises on any mismatch
    assert res["ok"]
    assert max(res["cd_rel_err_vs_f64_same_sketch"].values()) < 1e-5
