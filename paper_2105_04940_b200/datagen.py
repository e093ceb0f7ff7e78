"""Synthetic instances on the device -- SURVEY.md §8(f3), the reference's
``blockmm.datagen`` (pkg/src/blockmm/datagen.py:23-110).

Same names, arguments, validation errors and distributions: M's columns and
N's rows are i.i.d. N(0, Sigma) with the banded AR(1) covariance
Sigma_ij = scale * rho^|i-j| (or, heavy-tailed, location + z / sqrt(chi^2(1)):
multivariate t with one degree of freedom).  The reference draws on the host
and multiplies by a Cholesky factor; here ``bmm_gen_instance`` generates every
vector in HBM by the equivalent AR(1) recursion (csrc/datagen.cu), so an
instance costs one write of M and N and no host->device copy.

Deliberate difference: the random streams are this library's (PCG64 per
vector + Box-Muller), seeded from four 32-bit words drawn from ``rng``; the
instance is a deterministic function of (dims, rng state) like the
reference's, distribution-identical but not bit-identical to numpy's ziggurat
draws, and ``rng`` advances by those draws only.
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


def _generate(heavy: bool, m: int, n: int, p: int, rng: np.random.Generator, cov_left, cov_right, loc: float,
              device: bool, dtype):
    if min(m, n, p) < 1:
        raise ValueError("dimensions must be >= 1")
    cl, cr = _specs(m, p, cov_left, cov_right)
    tdt = torch.float32 if np.dtype(dtype) == np.float32 else torch.float64
    dev = _lib.device()
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
                        *, device: bool = False, dtype=np.float64):
    """M (m x n) with i.i.d. N(0, Sigma_left) columns, N (n x p) with i.i.d.
    N(0, Sigma_right) rows (datagen.py:55-72).  device=True keeps them in HBM."""
    return _generate(False, m, n, p, rng, cov_left, cov_right, 0.0, device, dtype)


def gen_heavy_tail_instance(m: int, n: int, p: int, rng: np.random.Generator,
                            cov_left: Optional[CovarianceSpec] = None, cov_right: Optional[CovarianceSpec] = None,
                            location: str = "ones", *, device: bool = False, dtype=np.float64):
    """location + z / sqrt(chi^2(1)) columns / rows (datagen.py:84-110)."""
    if min(m, n, p) < 1:
        raise ValueError("dimensions must be >= 1")
    if location not in ("ones", "zero"):
        raise ValueError("location must be 'ones' or 'zero'")
    return _generate(True, m, n, p, rng, cov_left, cov_right, 1.0 if location == "ones" else 0.0, device, dtype)
