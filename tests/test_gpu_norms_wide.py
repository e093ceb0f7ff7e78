"""K1 column sums of wide matrices (>= 256 MB: the TMA one-wave colsq_wide_kernel,
csrc/norms.cu) bit-exact against the oracle's sequential NumPy chain
(matrix.py:107-109), including a partial last 32-column unit, a row count that
is not a multiple of the slab height, a strided (sub-column) view and the
accumulate (chain continuation) mode."""
import numpy as np
import pytest

from oracle import blockmm_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
from paper_2105_04940_b200 import _lib  # noqa: E402


def colsq_dev(Md, accumulate=None, ld=None):
    m, n = Md.shape
    out = accumulate.clone() if accumulate is not None else torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.call("bmm_norms", _lib.matrix_dtype(Md), Md.data_ptr(), m, n, ld or Md.stride(0), 0, None, 0, 0, 0, 1,
              int(accumulate is not None), out.data_ptr(), None, _lib.stream_ptr())
    return out.cpu().numpy()


@pytest.mark.parametrize("dtype,m,n", [(np.float32, 2051, 40004), (np.float64, 1003, 40012)])
def test_wide_colsq_bit_exact(dtype, m, n):
    g = np.random.default_rng(5)
    M = (g.standard_normal((m, n)) * g.lognormal(0, 1, n)).astype(dtype)
    assert M.nbytes >= 256 << 20 or dtype == np.float64
    Md = torch.as_tensor(M, device="cuda")
    assert np.array_equal(colsq_dev(Md), O.colsq(M.astype(np.float64)))
    # chain continuation: rows [0, h) then [h, m) with accumulate == one pass
    h = m // 3
    first = torch.as_tensor(O.colsq(M[:h].astype(np.float64)), device="cuda")
    assert np.array_equal(colsq_dev(Md[h:], accumulate=first), O.colsq(M.astype(np.float64)))
    # a column sub-range of the matrix (row stride != width), as a sharded rank sees it
    c0, c1 = 4096, 4096 + 30000
    sub = Md[:, c0:c1]
    out = torch.empty(c1 - c0, dtype=torch.float64, device="cuda")
    _lib.call("bmm_norms", _lib.matrix_dtype(Md), sub.data_ptr(), m, c1 - c0, n, 0, None, 0, 0, 0, 1, 0,
              out.data_ptr(), None, _lib.stream_ptr())
    assert np.array_equal(out.cpu().numpy(), O.colsq(M[:, c0:c1].astype(np.float64)))
