"""Monte Carlo product estimators -- the reference's ``blockmm.estimators``
surface (pkg/src/blockmm/estimators.py) on the B200.

Per call: child streams are seeded on device from the caller's generator
(SeedSequence hashing + PCG64 in csrc/rng.cuh), the per-block CDFs are the
sequential cumsum, a warp per block draws its indices, the gather kernel
builds the rescaled sketch C (m x W) and D (W x p) bit-identically to
NumPy's ``Mb[:, idx] * scales``, and C @ D runs on the DMMA tensor pipe.
The caller-visible generator side effects (spawn counter / stream position)
are applied exactly as the reference leaves them.
"""
from __future__ import annotations

import csv
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np
import torch

from . import _lib
from . import rng as _rng
from .matrix import BlockPartition, device_gemm
from .plan import (
    BlockProbabilities,
    DeviceInstance,
    SamplingPlan,
    _check_instance,
    allocate_two_step,
    inst_block_q,
    optimal_probabilities,
    uniform_probabilities,
)


class DrawRecord(NamedTuple):
    """Per-draw audit trail of one sketch_columns call (estimators.py:47-52)."""

    columns: np.ndarray
    probs: np.ndarray
    scales: np.ndarray


@dataclass(frozen=True, eq=False)
class SketchPair:
    """Concatenated sketch factors; offsets[k]:offsets[k+1] is block k's slice
    of C's columns / D's rows (estimators.py:84-95)."""

    C: object
    D: object
    offsets: np.ndarray

    def block_product(self, k: int):
        lo, hi = int(self.offsets[k]), int(self.offsets[k + 1])
        out = device_gemm(_lib.to_device(self.C[:, lo:hi]), _lib.to_device(self.D[lo:hi, :]))
        return out if isinstance(self.C, torch.Tensor) else _lib.host(out)


@dataclass(frozen=True, eq=False)
class SampleLog:
    """Flat per-draw log across blocks; columns are global inner indices
    (estimators.py:98-116)."""

    block: np.ndarray
    draw: np.ndarray
    column: np.ndarray
    prob: np.ndarray
    scale: np.ndarray

    def __len__(self) -> int:
        return int(self.block.size)

    def write_csv(self, path, rep: int = 0) -> None:
        with open(path, "w", newline="") as fh:
            out = csv.writer(fh, lineterminator="\n")
            out.writerow(["rep", "block", "draw", "column_index", "probability", "scale"])
            for b, d, i, p, s in zip(self.block, self.draw, self.column, self.prob, self.scale):
                out.writerow([rep, int(b), int(d), int(i), f"{p:.17g}", f"{s:.17g}"])


class TwoStepResult(NamedTuple):
    pair: SketchPair
    product: object
    log: SampleLog
    plan: SamplingPlan


class BlockDrawRecord(NamedTuple):
    """Whole-block baseline audit trail (estimators.py:213-218)."""

    blocks: np.ndarray
    probs: np.ndarray
    scales: np.ndarray


# ---------------------------------------------------------------- device steps

def _u64_tensor(words: np.ndarray) -> torch.Tensor:
    return torch.as_tensor(np.asarray(words, dtype=np.uint64).view(np.int64), device=_lib.device())


def sample_blocks(inst: DeviceInstance, probs, budgets: np.ndarray, words: np.ndarray, first: int,
                  states: Optional[torch.Tensor] = None):
    """K3 on one instance: CDFs, child-stream seeding, draws.

    Returns device (column, prob, scale, col_off).  `states` overrides the
    spawned child streams (used for the caller's own stream)."""
    dev = _lib.device()
    K, n = inst.K, inst.n
    pr = probs if isinstance(probs, torch.Tensor) else _lib.f64(probs)
    cum = torch.empty(n, dtype=torch.float64, device=dev)
    last = torch.empty(K, dtype=torch.int64, device=dev)
    _lib.call("bmm_block_cdf", _lib.ptr(pr), _lib.ptr(inst.offsets), K, 1, n, _lib.ptr(cum),
              _lib.ptr(last), _lib.stream_ptr())
    budgets = np.asarray(budgets, dtype=np.int64)
    col_off_h = np.zeros(K + 1, dtype=np.int64)
    np.cumsum(budgets, out=col_off_h[1:])
    W = int(col_off_h[-1])
    bud_d = _lib.i64(budgets)
    col_off = _lib.i64(col_off_h)
    if states is None:
        states = torch.empty(4 * K, dtype=torch.int64, device=dev)
        words_d = torch.as_tensor(np.asarray(words, dtype=np.uint32).view(np.int32), device=dev)
        first_d = _lib.i64([first])
        _lib.call("bmm_seed_streams", _lib.ptr(words_d), int(len(words)), _lib.ptr(first_d), K, 1,
                  _lib.ptr(states), _lib.stream_ptr())
    column = torch.empty(max(W, 1), dtype=torch.int64, device=dev)
    prob = torch.empty(max(W, 1), dtype=torch.float64, device=dev)
    scale = torch.empty(max(W, 1), dtype=torch.float64, device=dev)
    max_len = int(getattr(inst, "max_len", n))
    _lib.call("bmm_sample", _lib.ptr(pr), _lib.ptr(cum), _lib.ptr(last), _lib.ptr(inst.offsets), K, 1, n, max_len,
              _lib.ptr(bud_d), _lib.ptr(col_off), W, _lib.ptr(states), _lib.ptr(column), _lib.ptr(prob),
              _lib.ptr(scale), _lib.stream_ptr())
    return column[:W], prob[:W], scale[:W], col_off


def gather_sketch(inst: DeviceInstance, column: torch.Tensor, scale: torch.Tensor, W: int,
                  dtype=torch.float64):
    """K4: C = M[:, column] * scale, D = N[column, :] * scale[:, None]."""
    M, N = inst.M, inst.N
    m, p = M.shape[0], N.shape[1]
    dev = M.device
    C = torch.empty((m, W), dtype=dtype, device=dev)
    D = torch.empty((W, p), dtype=dtype, device=dev)
    _lib.call("bmm_gather", _lib.matrix_dtype(M), _lib.matrix_dtype(C), _lib.ptr(M), M.stride(0), 0,
              _lib.ptr(N), N.stride(0), 0,
              m, p, _lib.ptr(column), _lib.ptr(scale), W, W, 1, _lib.ptr(C), W, 0, _lib.ptr(D), p, 0,
              _lib.stream_ptr())
    return C, D


def _out(t, as_numpy):
    return _lib.host(t) if as_numpy else t


# ---------------------------------------------------------------- public API

def sketch_columns(Mb, Nb, count: int, probs, rng: np.random.Generator):
    """Sample `count` rescaled column/row pairs of one block from the caller's
    stream (estimators.py:55-81)."""
    if Mb.ndim != 2 or Nb.ndim != 2 or Mb.shape[1] != Nb.shape[0]:
        raise ValueError(f"factor shapes do not chain: {tuple(Mb.shape)} x {tuple(Nb.shape)}")
    count = int(count)
    if count < 1:
        raise ValueError("count must be >= 1")
    pv = np.asarray(probs, dtype=np.float64)
    if pv.shape != (Mb.shape[1],):
        raise ValueError("need one probability per column")
    if (pv < 0).any() or abs(pv.sum() - 1.0) > 1e-9:
        raise ValueError("probabilities must be >= 0 and sum to 1")
    if not (pv > 0).any():
        raise ValueError("probability vector has empty support")
    part = BlockPartition((int(Mb.shape[1]),))
    inst = DeviceInstance(Mb, Nb, part)
    st = _u64_tensor(_rng.stream_state(rng))
    column, prob, scale, _ = sample_blocks(inst, pv, np.array([count]), None, 0, states=st)
    _rng.consume(rng, count)
    C, D = gather_sketch(inst, column, scale, count)
    as_np = _lib.want_numpy(Mb, Nb)
    rec = DrawRecord(_lib.host(column), _lib.host(prob), _lib.host(scale))
    return _out(C, as_np), _out(D, as_np), rec


def estimate_product(M, N, plan: SamplingPlan, rng: np.random.Generator):
    """Blocked importance-sampling estimate of M @ N under `plan`
    (estimators.py:125-175; Algorithm 2).  Returns (SketchPair, C @ D, SampleLog)."""
    part = plan.partition
    inst = DeviceInstance(M, N, part)
    K = part.num_blocks
    words, first = _rng.spawn_words(rng, K)
    budgets = plan.budgets
    column, prob, scale, col_off = sample_blocks(inst, plan.probs.flat(), budgets, words, first)
    W = int(plan.total)
    C, D = gather_sketch(inst, column, scale, W)
    CD = device_gemm(C, D)
    as_np = _lib.want_numpy(M, N)
    blocks = np.repeat(np.arange(K, dtype=np.int64), budgets)
    draws = np.concatenate([np.arange(int(b), dtype=np.int64) for b in budgets]) if W else np.zeros(0, np.int64)
    log = SampleLog(blocks, draws, _lib.host(column), _lib.host(prob), _lib.host(scale))
    pair = SketchPair(_out(C, as_np), _out(D, as_np), _lib.host(col_off))
    return pair, _out(CD, as_np), log


def estimate_product_two_step(M, N, part: BlockPartition, c: int, c0: int, rng: np.random.Generator,
                              pilot: str = "uniform", cap: bool = True) -> TwoStepResult:
    """Pilot block sizes, then estimate (estimators.py:185-210; Algorithm 3)."""
    if pilot == "uniform":
        p0 = uniform_probabilities(part)
    elif pilot == "norm":
        p0 = optimal_probabilities(M, N, part)
    else:
        raise ValueError(f"unknown pilot rule {pilot!r} (use 'uniform' or 'norm')")
    pilot_rng, main_rng = rng.spawn(2)
    plan = allocate_two_step(M, N, part, c, c0, p0, pilot_rng, cap=cap)
    pair, product, log = estimate_product(M, N, plan, main_rng)
    return TwoStepResult(pair, product, log, plan)


def estimate_product_block_sampling(M, N, part: BlockPartition, draws: int, rng: np.random.Generator,
                                    probs=None):
    """Whole-block baseline, tag SSM (estimators.py:221-253; Eq. 1.4)."""
    inst = DeviceInstance(M, N, part)
    K = part.num_blocks
    if probs is None:
        q, st = inst_block_q(inst)
        if st != _lib.ST_OK:
            raise ValueError("all blocks have zero norm: nothing to sample")
        q_host = _lib.host(q)
    else:
        q_host = np.asarray(probs, dtype=np.float64)
        if q_host.shape != (K,) or (q_host < 0).any() or abs(q_host.sum() - 1.0) > 1e-9:
            raise ValueError("block probabilities must be >= 0 and sum to 1")
        q = _lib.f64(q_host)
    draws = int(draws)
    if draws < 1:
        raise ValueError("draws must be >= 1")
    if not (q_host > 0).any():
        raise ValueError("probability vector has empty support")
    # one "block" spanning the K block probabilities, drawn from the caller's stream
    qinst = _BlockLevel(K)
    st = _u64_tensor(_rng.stream_state(rng))
    idx, qp, scale, _ = sample_blocks(qinst, q, np.array([draws]), None, 0, states=st)
    _rng.consume(rng, draws)
    idx_h = _lib.host(idx)
    widths = np.asarray(part.sizes, dtype=np.int64)[idx_h]
    sk_off = np.zeros(draws + 1, dtype=np.int64)
    np.cumsum(widths, out=sk_off[1:])
    W = int(sk_off[-1])
    M64, N64 = inst.M, inst.N
    if M64.dtype != torch.float64:
        M64, N64 = M64.to(torch.float64), N64.to(torch.float64)
    m, p = M64.shape[0], N64.shape[1]
    dev = M64.device
    C = torch.empty((m, W), dtype=torch.float64, device=dev)
    D = torch.empty((W, p), dtype=torch.float64, device=dev)
    sk_d = _lib.i64(sk_off)
    _lib.call("bmm_gather_blocks", _lib.BMM_F64, _lib.ptr(M64), M64.stride(0), _lib.ptr(N64), N64.stride(0),
              m, p, _lib.ptr(inst.offsets), _lib.ptr(idx), _lib.ptr(scale), _lib.ptr(sk_d), draws, W,
              _lib.ptr(C), W, _lib.ptr(D), p, _lib.stream_ptr())
    CD = device_gemm(C, D)
    as_np = _lib.want_numpy(M, N)
    rec = BlockDrawRecord(idx_h, _lib.host(qp), _lib.host(scale))
    return SketchPair(_out(C, as_np), _out(D, as_np), sk_off), _out(CD, as_np), rec


class _BlockLevel:
    """Minimal instance view for sampling over the K block probabilities."""

    def __init__(self, K: int):
        self.K = 1
        self.n = K
        self.max_len = K
        self.offsets = _lib.i64([0, K])
