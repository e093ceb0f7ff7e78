"""Synthetic instances on the device -- SURVEY.md §8(f3), the reference's
``blockmm.datagen`` (pkg/src/blockmm/datagen.py:23-110).

Same names, arguments, validation errors and distributions: M's columns and
N's rows are i.i.d. N(0, Sigma) with the banded AR(1) covariance
Sigma_ij = scale * rho^|i-j| (or, heavy-tailed, location + z / sqrt(chi^2(1)):
multivariate t with one degree of freedom).  The reference draws on the host
and multiplies by a Cholesky factor; here ``bmm_gen_instance`` generates every
vector in HBM by the equivalent AR(1) recursion (csrc/datagen.cu), so an
instance costs one write of M and N and no host->device copy.

Two stream modes:

* ``stream="numpy"`` (default, the drop-in): the variates are the reference's
  own -- ``rng.standard_normal`` / ``rng.chisquare`` called on the caller's
  Generator in the reference's order and shapes (datagen.py:70-71, 104-106), so
  the instance is the same pure function of (dims, rng state) and ``rng`` is
  left in exactly the reference's state.  numpy's ziggurat and gamma samplers
  are third-party arithmetic whose values depend on the host libm (log1p, pow),
  so they are not restated on the device; the variates are uploaded and
  ``bmm_ar1_transform`` replaces the Cholesky products ``L @ Z`` -- the only
  O(dim^2) work, 8 s of the reference's time at 1000 x 100000 -- by the
  recursion.  Entries agree with the reference's to BLAS rounding (1e-13 of the
  vector's norm; tests/golden/datagen.npz), the heavy-tailed division and
  location are applied in the reference's operation order.
* ``stream="device"``: this library's streams (PCG64 per vector + Box-Muller,
  seeded from four 32-bit words drawn from ``rng``), generated in HBM with no
  host traffic: distribution-identical, deterministic per seed, not the
  reference's values; ``rng`` advances by those four draws only.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib


@dataclass(frozen=True)
class CovarianceSpec:
    """datagen.py:23-35."""

    dim: int
    scale: float = 1.0
    rho: float = 0.7

    def __post_init__(self):
        if self.dim < 1:
            raise ValueError("dim must be >= 1")
        if self.scale <= 0:
            raise ValueError("scale must be > 0")
        if not -1.0 < self.rho < 1.0:
            raise ValueError("rho must lie in (-1, 1)")


def ar_covariance(spec: CovarianceSpec) -> np.ndarray:
    """scale * rho^|i-j| (datagen.py:38-42); a small host matrix for checks."""
    idx = np.arange(spec.dim)
    return spec.scale * spec.rho ** np.abs(idx[:, None] - idx[None, :])


def _specs(m: int, p: int, cov_left, cov_right):
    """datagen.py:45-52 defaults: left (1.0, 0.7), right (2.0, 0.7)."""
    cov_left = cov_left if cov_left is not None else CovarianceSpec(m, scale=1.0, rho=0.7)
    cov_right = cov_right if cov_right is not None else CovarianceSpec(p, scale=2.0, rho=0.7)
    if cov_left.dim != m or cov_right.dim != p:
        raise ValueError("covariance dims must match m and p")
    return cov_left, cov_right


def _chi_square_1(rng: np.random.Generator, n: int) -> np.ndarray:
    """n chi-square(1) draws from the caller's Generator with exact zeros redrawn, in the
    reference's call sequence (datagen.py:75-80: one more ``chisquare(1, #zeros)`` call per
    round, the new values filling the zero positions in ascending order), so the generator
    ends in the reference's state."""
    w = rng.chisquare(1.0, n)
    bad = np.flatnonzero(w == 0.0)
    while bad.size:
        w[bad] = rng.chisquare(1.0, bad.size)
        bad = bad[w[bad] == 0.0]
    return w


def _ar1(Z: np.ndarray, spec: CovarianceSpec, w, loc: float, transpose: bool, tdt) -> torch.Tensor:
    """L @ Z (datagen.py:70-71) on the device: Z is (dim, count); returns (dim, count) or its
    transpose (count, dim), heavy-tailed when w is given."""
    dim, count = Z.shape
    Zd = _lib.f64(Z)
    wd = _lib.f64(w) if w is not None else None
    out = torch.empty((count, dim) if transpose else (dim, count), dtype=tdt, device=_lib.device())
    _lib.call("bmm_ar1_transform", _lib.matrix_dtype(out), _lib.ptr(Zd), dim, count, count, int(transpose),
              float(spec.scale), float(spec.rho), _lib.ptr(wd), float(loc), _lib.ptr(out), out.shape[1],
              _lib.stream_ptr())
    return out


def _generate(heavy: bool, m: int, n: int, p: int, rng: np.random.Generator, cov_left, cov_right, loc: float,
              device: bool, dtype, stream: str = "numpy"):
    if min(m, n, p) < 1:
        raise ValueError("dimensions must be >= 1")
    if stream not in ("numpy", "device"):
        raise ValueError("stream must be 'numpy' or 'device'")
    cl, cr = _specs(m, p, cov_left, cov_right)
    tdt = torch.float32 if np.dtype(dtype) == np.float32 else torch.float64
    dev = _lib.device()
    if stream == "numpy":
        # the reference's draw order: Z_left, (w_left), Z_right, (w_right)
        Z = rng.standard_normal((m, n))
        w = _chi_square_1(rng, n) if heavy else None
        M = _ar1(Z, cl, w, loc, False, tdt)
        Z = rng.standard_normal((p, n))
        w = _chi_square_1(rng, n) if heavy else None
        N = _ar1(Z, cr, w, loc, True, tdt)
        del Z
        return (M, N) if device else (_lib.host(M), _lib.host(N))
    w = rng.integers(0, 2 ** 32, size=4, dtype=np.uint64)
    seed_lo = int(w[0]) | (int(w[1]) << 32)
    seed_hi = int(w[2]) | (int(w[3]) << 32)
    M = torch.empty((m, n), dtype=tdt, device=dev)
    N = torch.empty((n, p), dtype=tdt, device=dev)
    _lib.call("bmm_gen_instance", int(heavy), _lib.matrix_dtype(M), m, n, p, seed_hi, seed_lo, float(cl.scale),
              float(cl.rho), float(cr.scale), float(cr.rho), float(loc), _lib.ptr(M), n, _lib.ptr(N), p,
              _lib.stream_ptr())
    if device:
        return M, N
    return _lib.host(M), _lib.host(N)


def gen_normal_instance(m: int, n: int, p: int, rng: np.random.Generator,
                        cov_left: Optional[CovarianceSpec] = None, cov_right: Optional[CovarianceSpec] = None,
                        *, device: bool = False, dtype=np.float64, stream: str = "numpy"):
    """M (m x n) with i.i.d. N(0, Sigma_left) columns, N (n x p) with i.i.d.
    N(0, Sigma_right) rows (datagen.py:55-72).  device=True keeps them in HBM."""
    return _generate(False, m, n, p, rng, cov_left, cov_right, 0.0, device, dtype, stream)


def gen_heavy_tail_instance(m: int, n: int, p: int, rng: np.random.Generator,
                            cov_left: Optional[CovarianceSpec] = None, cov_right: Optional[CovarianceSpec] = None,
                            location: str = "ones", *, device: bool = False, dtype=np.float64,
                            stream: str = "numpy"):
    """location + z / sqrt(chi^2(1)) columns / rows (datagen.py:84-110)."""
    if min(m, n, p) < 1:
        raise ValueError("dimensions must be >= 1")
    if location not in ("ones", "zero"):
        raise ValueError("location must be 'ones' or 'zero'")
    return _generate(True, m, n, p, rng, cov_left, cov_right, 1.0 if location == "ones" else 0.0, device, dtype,
                     stream)
