"""The summation orders the device kernels restate (csrc/pairwise.cuh, norms.cu,
sample.cu) checked against numpy with pure-Python loops.  CPU only."""
import numpy as np

import oracle.blockmm_oracle as O


def pairwise(a):
    n = len(a)
    if n < 8:
        r = 0.0
        for x in a:
            r = r + x
        return r
    if n <= 128:
        r = list(a[:8])
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] = r[j] + a[i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for x in a[i:]:
            res = res + x
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise(a[:n2]) + pairwise(a[n2:])


def test_pairwise_sum_and_reduceat():
    g = np.random.default_rng(0)
    for n in list(range(1, 140)) + [255, 256, 257, 500, 1000, 4096, 16384, 20000]:
        a = g.standard_normal(n) ** 2 * g.lognormal(0, 3, n)
        assert pairwise(a) == a.sum()
        assert np.add.reduceat(a, [0])[0] == (a[0] + pairwise(a[1:]) if n > 1 else a[0])


def test_row_norm_is_pairwise_and_col_norm_sequential():
    g = np.random.default_rng(1)
    N = g.standard_normal((5, 300)) * g.lognormal(0, 2, (5, 300))
    rs = O.rowsq(N)
    for i in range(5):
        assert rs[i] == pairwise(N[i] * N[i])
    M = g.standard_normal((77, 9)) * g.lognormal(0, 2, (77, 9))
    acc = np.zeros(9)
    for h in range(77):
        acc = acc + M[h] * M[h]
    assert np.array_equal(O.colsq(M), acc)
    assert np.array_equal(np.linalg.norm(M, axis=0), np.sqrt(acc))


def test_chunked_colsq_is_exact():
    g = np.random.default_rng(2)
    M = g.standard_normal((1000, 64)).astype(np.float32)
    assert np.array_equal(O.colsq_chunked(M, rows=37), O.colsq(M.astype(np.float64)))


def test_cumsum_sequential():
    g = np.random.default_rng(3)
    a = g.random(1000)
    acc, out = 0.0, []
    for x in a:
        acc = acc + x
        out.append(acc)
    assert np.cumsum(a).tolist() == out
