"""Pilot norms ||C0_k D0_k||_F^2 by Gram matrices (bmm_segsq_gram_gather) against
the DMMA kernel (bmm_segsq_f64_gather) and NumPy on the gathered sketch
(plan.py:457-464): segment lengths 0..20 (1-3 Gram tiles), float32 inputs,
batches.  Tolerance 1e-13 relative (BLAS order differs)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(M, N, col, sc, seg):
    C = M[:, col] * sc
    D = N[col, :] * sc[:, None]
    out = []
    for j in range(len(seg) - 1):
        P = C[:, seg[j]:seg[j + 1]] @ D[seg[j]:seg[j + 1]]
        out.append(float(np.sum(P * P)))
    return np.array(out)


def _gram(M, N, col, sc, seg, dtype=np.float64, batch=1, max_len=None):
    from paper_2105_04940_b200 import _lib
    Md = torch.as_tensor(np.ascontiguousarray(M.astype(dtype)), device="cuda")
    Nd = torch.as_tensor(np.ascontiguousarray(N.astype(dtype)), device="cuda")
    m, n = M.shape[-2:]
    p = N.shape[-1]
    K = seg.shape[-1] - 1
    W = col.shape[-1]
    cd, sd, gd = _lib.i64(col.ravel()), torch.as_tensor(sc.ravel(), device="cuda"), _lib.i64(seg.ravel())
    out = torch.empty(batch * K, dtype=torch.float64, device="cuda")
    _lib.call("bmm_segsq_gram_gather", _lib.matrix_dtype(Md), Md.data_ptr(), n, m * n if batch > 1 else 0,
              Nd.data_ptr(), p, n * p if batch > 1 else 0, m, p, cd.data_ptr(), sd.data_ptr(), W, gd.data_ptr(), K,
              K + 1, int(np.diff(seg, axis=-1).max()) if max_len is None else max_len, batch, out.data_ptr(),
              _lib.stream_ptr())
    return out.cpu().numpy().reshape(batch, K) if batch > 1 else out.cpu().numpy()


def _case(g, m, n, p, lens):
    M = g.standard_normal((m, n)) * g.lognormal(0, 1, n)
    N = g.standard_normal((n, p)) * g.lognormal(0, 1, (n, 1))
    W = int(sum(lens))
    col = g.integers(0, n, W)
    sc = 1.0 / np.sqrt(g.uniform(0.01, 1.0, W) * 7)
    seg = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return M, N, col, sc, seg


@pytest.mark.parametrize("m,n,p", [(1, 30, 1), (24, 500, 16), (300, 2000, 257), (1000, 4000, 1000)])
def test_gram_matches_numpy(m, n, p):
    g = np.random.default_rng(m + p)
    lens = [0, 1, 2, 5, 7, 8, 9, 16, 17, 20, 5, 5, 3]
    M, N, col, sc, seg = _case(g, m, n, p, lens)
    got = _gram(M, N, col, sc, seg)
    ref = _ref(M, N, col, sc, seg)
    assert got[0] == 0.0
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=0)


def test_gram_matches_dmma_float32_and_batch():
    from paper_2105_04940_b200 import _lib
    g = np.random.default_rng(3)
    m, n, p = 200, 1000, 150
    M, N, col, sc, seg = _case(g, m, n, p, [5] * 40)
    M32, N32 = M.astype(np.float32), N.astype(np.float32)
    got = _gram(M32, N32, col, sc, seg, dtype=np.float32)
    np.testing.assert_allclose(got, _ref(M32.astype(np.float64), N32.astype(np.float64), col, sc, seg), rtol=1e-13)
    # the DMMA kernel on the same sketch
    Md, Nd = torch.as_tensor(M, device="cuda"), torch.as_tensor(N, device="cuda")
    K = len(seg) - 1
    cd, sd, gd = _lib.i64(col), torch.as_tensor(sc, device="cuda"), _lib.i64(seg)
    dm = torch.empty(K, dtype=torch.float64, device="cuda")
    ws = _lib.workspace(_lib.load().bmm_segsq_f64_workspace(m, p, K, 1))
    _lib.call("bmm_segsq_f64_gather", Md.data_ptr(), n, 0, Nd.data_ptr(), p, 0, m, p, cd.data_ptr(), sd.data_ptr(),
              len(col), gd.data_ptr(), K, 0, 1, dm.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    np.testing.assert_allclose(_gram(M, N, col, sc, seg), dm.cpu().numpy(), rtol=1e-13)
    # batch of 3 problems with their own sketches
    Ms = np.stack([M, 2 * M, M[::-1].copy()])
    Ns = np.stack([N, N[:, ::-1].copy(), 0.5 * N])
    cols = np.stack([col, col[::-1].copy(), col])
    scs = np.stack([sc, sc, 3 * sc])
    segs = np.stack([seg, seg, seg])
    got = _gram(Ms, Ns, cols, scs, segs, batch=3)
    for b in range(3):
        np.testing.assert_allclose(got[b], _ref(Ms[b], Ns[b], cols[b], scs[b], seg), rtol=1e-13)
