"""Factor matrices, the inner-dimension block partition, norms and the exact
product -- the reference's ``blockmm.matrix`` surface
(pkg/src/blockmm/matrix.py:21-118) computed on the B200.

Inputs may be NumPy arrays (copied to the device; NumPy results are returned)
or CUDA tensors (device-resident; CUDA tensors are returned).  float32 inputs
are accepted and accumulated in float64, which equals the reference run on
the float64-upcast matrices.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


def as_matrix(values) -> np.ndarray:
    """float64 C-ordered 2-D matrix with finite entries (matrix.py:21-32).

    Host-side input validation only; it is what the reference uses to coerce
    user data before any arithmetic."""
    a = np.ascontiguousarray(values, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={a.ndim}")
    if not np.isfinite(a).all():
        raise ValueError("matrix contains NaN or Inf entries")
    return a


@dataclass(frozen=True)
class BlockPartition:
    """K contiguous blocks of the shared inner dimension (matrix.py:35-79)."""

    sizes: tuple

    def __post_init__(self):
        sz = tuple(int(s) for s in self.sizes)
        if not sz:
            raise ValueError("partition needs at least one block")
        if min(sz) < 1:
            raise ValueError(f"every block size must be >= 1, got {sz}")
        object.__setattr__(self, "sizes", sz)

    @classmethod
    def equal(cls, n: int, num_blocks: int) -> "BlockPartition":
        if num_blocks < 1 or n % num_blocks:
            raise ValueError(f"n={n} is not divisible into {num_blocks} equal blocks")
        return cls((n // num_blocks,) * num_blocks)

    @property
    def num_blocks(self) -> int:
        return len(self.sizes)

    @property
    def total(self) -> int:
        return int(sum(self.sizes))

    @property
    def offsets(self) -> np.ndarray:
        out = np.zeros(len(self.sizes) + 1, dtype=np.int64)
        np.cumsum(self.sizes, out=out[1:])
        return out

    def block_slice(self, k: int) -> slice:
        if k < 0 or k >= len(self.sizes):
            raise IndexError(f"block index {k} out of range for K={len(self.sizes)}")
        start = sum(self.sizes[:k])
        return slice(start, start + self.sizes[k])

    def check_length(self, length: int, what: str = "axis") -> None:
        if self.total != length:
            raise ValueError(f"partition covers {self.total} indices but {what} has length {length}")


def block_view(M, part: BlockPartition, k: int, axis: str = "columns"):
    """Zero-copy block k of M: columns of the left factor or rows of the
    right factor (matrix.py:82-95)."""
    sl = part.block_slice(k)
    if axis == "columns":
        part.check_length(M.shape[1], "column axis")
        return M[:, sl]
    if axis == "rows":
        part.check_length(M.shape[0], "row axis")
        return M[sl, :]
    raise ValueError(f"axis must be 'columns' or 'rows', got {axis!r}")


# ---------------------------------------------------------------- device ops

def device_norms_sq(Md: torch.Tensor | None, Nd: torch.Tensor | None):
    """K1: (colsq of M, rowsq of N) as float64 CUDA vectors."""
    colsq = rowsq = None
    src = Md if Md is not None else Nd
    dtype = _lib.matrix_dtype(src)
    if Md is not None and Nd is not None and Md.dtype != Nd.dtype:
        Nd = Nd.to(Md.dtype)
    m, n = (Md.shape if Md is not None else (0, Nd.shape[0]))
    p = Nd.shape[1] if Nd is not None else 0
    dev = src.device
    if Md is not None:
        colsq = torch.empty(n, dtype=torch.float64, device=dev)
    if Nd is not None:
        rowsq = torch.empty(Nd.shape[0], dtype=torch.float64, device=dev)
    _lib.call("bmm_norms", dtype,
              _lib.ptr(Md), m, n, Md.stride(0) if Md is not None else 0, 0,
              _lib.ptr(Nd), p, Nd.stride(0) if Nd is not None else 0, 0,
              1, 0, _lib.ptr(colsq), _lib.ptr(rowsq), _lib.stream_ptr())
    return colsq, rowsq


def device_pairwise_sum(x: torch.Tensor) -> torch.Tensor:
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    _lib.call("bmm_pairwise_sum", _lib.ptr(x), x.numel(), x.numel(), 1, _lib.ptr(out), _lib.stream_ptr())
    return out


def device_gemm(Ad: torch.Tensor, Bd: torch.Tensor) -> torch.Tensor:
    """K5/K8: float64 A @ B on the DMMA pipe (float32 operands are upcast)."""
    if Ad.dtype != torch.float64:
        Ad = Ad.to(torch.float64)
    if Bd.dtype != torch.float64:
        Bd = Bd.to(torch.float64)
    m, k = Ad.shape
    nc = Bd.shape[1]
    out = torch.empty((m, nc), dtype=torch.float64, device=Ad.device)
    wsb = _lib.load().bmm_gemm_f64_workspace(m, nc, k, 1)
    ws = _lib.workspace(wsb)
    _lib.call("bmm_gemm_f64", _lib.ptr(Ad), Ad.stride(0), 0, _lib.ptr(Bd), Bd.stride(0), 0,
              m, nc, k, 1, _lib.ptr(out), nc, 0, _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    return out


def _ret(t: torch.Tensor, as_numpy: bool):
    return _lib.host(t) if as_numpy else t


# ---------------------------------------------------------------- public API

def multiply_exact(M, N):
    """Exact product MN (matrix.py:98-104), float64 DMMA GEMM on device."""
    if M.ndim != 2 or N.ndim != 2:
        raise ValueError("both factors must be 2-D")
    if M.shape[1] != N.shape[0]:
        raise ValueError(f"inner dimensions differ: {M.shape} x {N.shape}")
    out = device_gemm(_lib.float_matrix(M), _lib.float_matrix(N))
    return _ret(out, _lib.want_numpy(M, N))


def column_norms(M):
    """Euclidean norm of each column (matrix.py:107-109)."""
    colsq, _ = device_norms_sq(_lib.float_matrix(M), None)
    return _ret(torch.sqrt(colsq), _lib.want_numpy(M))


def row_norms(N):
    """Euclidean norm of each row (matrix.py:112-114)."""
    _, rowsq = device_norms_sq(None, _lib.float_matrix(N))
    return _ret(torch.sqrt(rowsq), _lib.want_numpy(N))


def frobenius_norm(M) -> float:
    """||M||_F (matrix.py:117-118): pairwise sum of the column sums of squares."""
    Md = _lib.float_matrix(M)
    if Md.ndim == 1:
        Md = Md.reshape(1, -1)
    colsq, _ = device_norms_sq(Md, None)
    return float(torch.sqrt(device_pairwise_sum(colsq)).item())


def __getattr__(name):
    """The reference defines its matrix file formats in matrix.py (121-140); here
    they live in io.py.  Resolve them lazily (io imports this module)."""
    if name in ("load_matrix", "load_matrix_csv", "save_matrix", "save_matrix_csv"):
        from . import io
        return getattr(io, name)
    raise AttributeError(name)
