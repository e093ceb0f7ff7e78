"""Exact variance analytics -- SURVEY.md §8(f2), the reference's
``elementwise_variance`` / ``expected_sq_error`` / ``minimum_expected_sq_error``
(pkg/src/blockmm/analysis.py:57-125) on the B200.

elementwise_variance: the reference loops over blocks forming
(M_k^2 / p) @ N_k^2 and (M_k N_k)^2 per block.  Here the first term is ONE
squared-mode DMMA GEMM over the whole inner dimension with per-column weights
1/(c_k p_i), and the second a segmented GEMM whose epilogue accumulates
(M^k N_k)^2 / c_k into the output tile (bmm_elementwise_variance).
expected_sq_error: per-block sums of sc_i^2/p_i (bmm_block_term1) and the
segmented square sums g_k^2 (bmm_segsq_f64); only the K-term loop of the
reference runs on the host.  Results agree with the reference to rounding
(BLAS order there, DMMA order here); the validation errors are the
reference's, raised in the reference's block order.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .matrix import BlockPartition, device_gemm
from .plan import DeviceInstance, SamplingPlan, _check_instance, optimal_size_weights


def _block_budgets(plan: SamplingPlan, budgets) -> np.ndarray:
    """analysis.py:46-54."""
    if budgets is None:
        return plan.budgets.astype(np.float64)
    b = np.asarray(budgets, dtype=np.float64)
    if b.shape != (plan.partition.num_blocks,) or (b < 0).any():
        raise ValueError("budget override must be one nonnegative value per block")
    return b


def _f64_instance(M, N, part) -> DeviceInstance:
    inst = DeviceInstance(M, N, part)
    if inst.M.dtype != torch.float64:  # the analytics kernels are float64 (reference: fp64 throughout)
        inst.M, inst.N = inst.M.to(torch.float64), inst.N.to(torch.float64)
    return inst


def _variance_device(inst: DeviceInstance, probs: torch.Tensor, budgets: np.ndarray):
    """(var m x p, first bad block or None) for a whole instance."""
    m, n, p, K = int(inst.M.shape[0]), inst.n, int(inst.N.shape[1]), inst.K
    colsq, rowsq = inst.norms
    var = torch.empty((m, p), dtype=torch.float64, device=inst.M.device)
    bad = torch.empty(1, dtype=torch.int64, device=inst.M.device)
    ws = _lib.workspace(_lib.load().bmm_variance_workspace(m, p, n, K))
    bud = _lib.f64(budgets)
    _lib.call("bmm_elementwise_variance", _lib.ptr(inst.M), inst.M.stride(0), _lib.ptr(inst.N), inst.N.stride(0),
              m, n, p, _lib.ptr(inst.offsets), K, _lib.ptr(probs), _lib.ptr(colsq), _lib.ptr(rowsq), _lib.ptr(bud),
              _lib.ptr(var), p, _lib.ptr(bad), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    b = int(bad.item())
    return var, (K - b if b else None)


def _zero_budget_blocks_ok(inst: DeviceInstance, plan: SamplingPlan, b: np.ndarray, upto: int) -> None:
    """Blocks k < upto with c_k = 0 must carry no sampling variance
    (analysis.py:83-87); raise the reference's error for the first that does."""
    part = plan.partition
    off = part.offsets
    for k in np.flatnonzero(b[:upto] == 0):
        k = int(k)
        lo, hi = int(off[k]), int(off[k + 1])
        sub = BlockPartition((hi - lo,))
        blk = DeviceInstance(inst.M[:, lo:hi].contiguous(), inst.N[lo:hi].contiguous(), sub)
        pk = _lib.f64(plan.probs[k])
        var1, _ = _variance_device(blk, pk, np.ones(1))  # term1 - exact^2 at c_k = 1
        exact_sq = device_gemm(blk.M, blk.N) ** 2
        term1 = var1 + exact_sq
        scale = max(1.0, float(term1.max().item()) if term1.numel() else 0.0)
        if float(var1.abs().max().item()) > 1e-12 * scale:
            raise ValueError(f"block {k}: zero budget on a block with sampling variance")


def elementwise_variance(M, N, plan: SamplingPlan, budgets=None):
    """Exact per-entry variance of the blocked estimate (analysis.py:57-90)."""
    part = plan.partition
    _check_instance(M, N, part)
    b = _block_budgets(plan, budgets)
    inst = _f64_instance(M, N, part)
    var, bad = _variance_device(inst, _lib.f64(plan.probs.flat()), b)
    _zero_budget_blocks_ok(inst, plan, b, part.num_blocks if bad is None else bad)
    if bad is not None:
        raise ValueError(f"block {bad}: zero probability at a contributing column")
    return _lib.host(var) if _lib.want_numpy(M, N) else var


def expected_sq_error(M, N, plan: SamplingPlan, budgets=None) -> float:
    """E ||MN - estimate||_F^2 in closed form (analysis.py:93-116)."""
    part = plan.partition
    _check_instance(M, N, part)
    b = _block_budgets(plan, budgets)
    inst = _f64_instance(M, N, part)
    K = inst.K
    colsq, rowsq = inst.norms
    term1_d = torch.empty(K, dtype=torch.float64, device=colsq.device)
    bad_d = torch.empty(1, dtype=torch.int64, device=colsq.device)
    probs = _lib.f64(plan.probs.flat())
    _lib.call("bmm_block_term1", _lib.ptr(probs), _lib.ptr(colsq), _lib.ptr(rowsq), _lib.ptr(inst.offsets), K,
              _lib.ptr(term1_d), _lib.ptr(bad_d), _lib.stream_ptr())
    g_sq = _lib.host(inst.block_product_sq())
    term1 = _lib.host(term1_d)
    badv = int(bad_d.item())
    bad = K - badv if badv else None
    total = 0.0
    for k in range(K):
        if bad is not None and k == bad:
            raise ValueError(f"block {k}: zero probability at a contributing column")
        numerator = float(term1[k]) - float(g_sq[k])
        if b[k] == 0:
            if abs(numerator) > 1e-12 * max(1.0, float(term1[k])):
                raise ValueError(f"block {k}: zero budget on a block with sampling variance")
            continue
        total += numerator / b[k]
    return total


def minimum_expected_sq_error(M, N, part: BlockPartition, c: int) -> float:
    """(sum_k sqrt(s_k^2 - g_k^2))^2 / c  (analysis.py:119-125)."""
    if c <= 0:
        raise ValueError("budget must be positive")
    w = optimal_size_weights(M, N, part)
    return float(w.sum() ** 2) / c
