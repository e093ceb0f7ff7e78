"""Error evaluation on the product estimate (K9).

relative_error mirrors pkg/src/blockmm/analysis.py:318-325
(||exact - approx||_F / ||exact||_F); product_error additionally returns the
BASELINE metric ||MN - CD||_F / (||M||_F ||N||_F).  Both reduce on device with
bmm_sqdiff (float64, fixed-order two-level reduction).
"""
from __future__ import annotations

import math

import torch

from . import _lib


def sq_diff(X, Y=None):
    """(sum (X - Y)^2, sum X^2) on device; Y=None gives (sum X^2, sum X^2)."""
    Xd = _lib.to_device(X)
    if Xd.dtype not in (torch.float64, torch.float32):
        Xd = Xd.to(torch.float64)
    Yd = None
    if Y is not None:
        Yd = _lib.to_device(Y)
        if Yd.dtype != Xd.dtype:
            Yd = Yd.to(Xd.dtype)
    if Xd.ndim == 1:
        Xd = Xd.reshape(1, -1)
        Yd = Yd.reshape(1, -1) if Yd is not None else None
    m, nc = Xd.shape
    out = torch.empty(2, dtype=torch.float64, device=Xd.device)
    ws = _lib.workspace(_lib.load().bmm_sqdiff_workspace(m, nc, 1))
    _lib.call("bmm_sqdiff", _lib.matrix_dtype(Xd), _lib.ptr(Xd), Xd.stride(0), 0, _lib.ptr(Yd),
              Yd.stride(0) if Yd is not None else 0, 0, m, nc, 1, _lib.ptr(out), _lib.ptr(ws), ws.numel(),
              _lib.stream_ptr())
    e, r = _lib.host(out)
    return float(e), float(r)


def relative_error(approx, exact) -> float:
    """||exact - approx||_F / ||exact||_F  (analysis.py:318-325)."""
    if tuple(approx.shape) != tuple(exact.shape):
        raise ValueError(f"shapes differ: {tuple(approx.shape)} vs {tuple(exact.shape)}")
    err, ref = sq_diff(exact, approx)
    if ref == 0.0:
        raise ValueError("exact matrix has zero norm")
    return math.sqrt(err) / math.sqrt(ref)
