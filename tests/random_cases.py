"""Random instances shared by the randomised sweeps (CPU oracle-vs-reference
and GPU-vs-oracle): random partitions (size-1 blocks, very unequal blocks),
heavy-tailed column/row scales, zeroed columns of M and a zeroed block of N."""
import numpy as np


def random_instance(g):
    K = int(g.integers(1, 24))
    kind = g.integers(0, 3)
    if kind == 0:
        sizes = g.integers(1, 40, K)
    elif kind == 1:
        sizes = np.maximum(1, (g.lognormal(3, 1.2, K)).astype(int))
    else:
        sizes = np.full(K, int(g.integers(1, 64)))
    n = int(sizes.sum())
    m, p = int(g.integers(1, 70)), int(g.integers(1, 70))
    M = g.standard_normal((m, n)) * g.lognormal(0, 1.5, n)
    N = g.standard_normal((n, p)) * g.lognormal(0, 1.5, (n, 1))
    if g.random() < 0.3:
        M[:, g.integers(0, n, max(1, n // 10))] = 0.0
    if g.random() < 0.2 and K > 1:
        k = int(g.integers(0, K))
        o = int(sizes[:k].sum())
        N[o:o + sizes[k]] = 0.0
    return M, N, tuple(int(s) for s in sizes)


def sweep_params(seed: int):
    """Instance + budget c (live <= c <= total caps) + pilot budget c0 (1-3 pilot
    draws per block) for sweep seed `seed`."""
    g = np.random.default_rng(1000 + seed)
    M, N, sizes = random_instance(g)
    K = len(sizes)
    off = np.concatenate([[0], np.cumsum(sizes)])
    cs = np.sum(M * M, axis=0)
    rs = np.sum(N * N, axis=1)
    live = sum(bool(np.any((cs[off[k]:off[k + 1]] > 0) & (rs[off[k]:off[k + 1]] > 0))) for k in range(K))
    caps = sum(sz for k, sz in enumerate(sizes)
               if np.any((cs[off[k]:off[k + 1]] > 0) & (rs[off[k]:off[k + 1]] > 0)))
    c = int(g.integers(max(live, 1), max(live, caps) + 1))
    c0 = K * int(g.integers(1, 4))
    return M, N, sizes, c, c0
