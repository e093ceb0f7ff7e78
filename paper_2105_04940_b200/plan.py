"""Sampling plans -- the reference's ``blockmm.plan`` hot-path surface
(pkg/src/blockmm/plan.py) with every numeric step on the B200:

* one K1 norm pass feeds probabilities, score sums and budgets (the reference
  recomputes the norms two or three times per allocator, plan.py:165-173);
* K2 (bmm_block_probs) gives the per-block probabilities and score sums in
  NumPy's exact summation order, so they are bit-identical;
* the block-product norms g_k of the optimal allocator come from the DMMA
  segmented square-sum GEMM (plan.py:183-188);
* integer budgets come from the device largest-remainder kernel
  (bmm_budgets, plan.py:242-347), bit-identical budgets for identical inputs.
The host only validates arguments, reads back results and builds the same
frozen records the reference returns.
"""
from __future__ import annotations

import os

import json
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np
import torch

from . import _lib
from . import rng as _rng
from .matrix import BlockPartition, device_norms_sq

METHOD_TAGS = ("OPL", "ONC", "ONU", "ONMCNR", "UU", "SSM")
PROB_SUM_TOL = 1e-12
RADICAND_SLACK = 1e-9


def _check_instance(M, N, part: BlockPartition) -> None:
    """plan.py:41-46."""
    if M.ndim != 2 or N.ndim != 2:
        raise ValueError("factors must be 2-D")
    if M.shape[1] != N.shape[0]:
        raise ValueError(f"inner dimensions differ: {M.shape} x {N.shape}")
    part.check_length(M.shape[1], "inner dimension")


@dataclass(frozen=True, eq=False)
class BlockProbabilities:
    """Per-block probability vectors (plan.py:49-99): each sums to 1 within
    PROB_SUM_TOL, or is all zero for a flagged zero-score block."""

    per_block: tuple
    rule: str = "explicit"

    def __post_init__(self):
        checked = []
        for k, vec in enumerate(self.per_block):
            v = np.ascontiguousarray(vec, dtype=np.float64)
            if v.ndim != 1 or v.size == 0:
                raise ValueError(f"block {k}: probabilities must be a nonempty vector")
            if not np.isfinite(v).all() or (v < 0).any():
                raise ValueError(f"block {k}: probabilities must be finite and >= 0")
            tot = v.sum()
            if tot != 0.0 and abs(tot - 1.0) > PROB_SUM_TOL:
                raise ValueError(f"block {k}: probabilities sum to {tot!r}, not 1")
            checked.append(v)
        object.__setattr__(self, "per_block", tuple(checked))

    def __len__(self) -> int:
        return len(self.per_block)

    def __getitem__(self, k: int) -> np.ndarray:
        return self.per_block[k]

    @property
    def num_blocks(self) -> int:
        return len(self.per_block)

    @property
    def zero_blocks(self) -> tuple:
        return tuple(k for k, v in enumerate(self.per_block) if v.sum() == 0.0)

    def check_partition(self, part: BlockPartition) -> None:
        if len(self.per_block) != part.num_blocks:
            raise ValueError(f"probabilities cover {len(self.per_block)} blocks, "
                             f"partition has {part.num_blocks}")
        for k, (v, nk) in enumerate(zip(self.per_block, part.sizes)):
            if v.size != nk:
                raise ValueError(f"block {k}: {v.size} probabilities for {nk} columns")

    def flat(self) -> np.ndarray:
        """All blocks concatenated in partition order (the device layout)."""
        return np.concatenate(self.per_block) if self.per_block else np.zeros(0)


@dataclass(frozen=True, eq=False)
class BlockScores:
    """Score sums s_k and block-product norms g_k (plan.py:102-122)."""

    score_sums: np.ndarray
    product_norms: np.ndarray
    exact: bool = True

    def __post_init__(self):
        s = np.asarray(self.score_sums, dtype=np.float64)
        g = np.asarray(self.product_norms, dtype=np.float64)
        if s.ndim != 1 or s.shape != g.shape:
            raise ValueError("score_sums and product_norms must be matching vectors")
        if (s < 0).any() or (g < 0).any():
            raise ValueError("scores must be nonnegative")
        if self.exact and (g > s * (1 + RADICAND_SLACK) + 1e-300).any():
            raise ValueError("exact product norm exceeds score sum (Cauchy-Schwarz violated)")
        object.__setattr__(self, "score_sums", s)
        object.__setattr__(self, "product_norms", g)


@dataclass(frozen=True, eq=False)
class SamplingPlan:
    """Partition + probabilities + integer budgets (plan.py:125-162)."""

    partition: BlockPartition
    probs: BlockProbabilities
    budgets: np.ndarray
    method: str = ""
    notes: tuple = ()
    pilot_norms: Optional[np.ndarray] = None

    def __post_init__(self):
        b = np.asarray(self.budgets)
        if b.dtype.kind not in "iu" and not np.array_equal(b, np.round(b)):
            raise ValueError("budgets must be integers")
        b = b.astype(np.int64)
        if b.ndim != 1 or b.size != self.partition.num_blocks:
            raise ValueError("budgets must be one integer per block")
        if (b < 0).any():
            raise ValueError("budgets must be >= 0")
        self.probs.check_partition(self.partition)
        zero = set(self.probs.zero_blocks)
        for k in range(self.partition.num_blocks):
            if (b[k] == 0) != (k in zero):
                raise ValueError(f"block {k}: zero budget and zero-probability flag must coincide")
        object.__setattr__(self, "budgets", b)
        if self.pilot_norms is not None:
            pn = np.asarray(self.pilot_norms, dtype=np.float64)
            if pn.shape != (self.partition.num_blocks,):
                raise ValueError("pilot_norms must be one value per block")
            object.__setattr__(self, "pilot_norms", pn)

    @property
    def total(self) -> int:
        return int(self.budgets.sum())


# ---------------------------------------------------------------- device core

class DeviceInstance:
    """Device copies of (M, N) plus the products of one K1 norm pass.

    Every plan / estimator entry point builds one of these, so a single norm
    pass feeds probabilities, score sums and budgets."""

    def __init__(self, M, N, part: BlockPartition):
        _check_instance(M, N, part)
        self.M = _lib.float_matrix(M)
        self.N = _lib.float_matrix(N)
        if self.N.dtype != self.M.dtype:
            self.N = self.N.to(torch.float64)
            self.M = self.M.to(torch.float64)
        self.part = part
        self.K = part.num_blocks
        self.n = int(self.M.shape[1])
        self.offsets = _lib.i64(part.offsets)
        self.sizes = _lib.i64(part.sizes)
        self.max_len = int(max(part.sizes))
        self._norms = None

    @property
    def norms(self):
        if self._norms is None:
            self._norms = device_norms_sq(self.M, self.N)
        return self._norms

    def block_stats(self, probs=True, s=True, fnorm=False):
        colsq, rowsq = self.norms
        dev = colsq.device
        pr = torch.empty(self.n, dtype=torch.float64, device=dev) if probs else None
        sk = torch.empty(self.K, dtype=torch.float64, device=dev) if s else None
        fk = torch.empty(self.K, dtype=torch.float64, device=dev) if fnorm else None
        _lib.call("bmm_block_probs", _lib.ptr(colsq), _lib.ptr(rowsq), self.n, _lib.ptr(self.offsets),
                  self.K, 1, self.max_len, _lib.ptr(pr), _lib.ptr(sk), _lib.ptr(fk), None, None, _lib.stream_ptr())
        return pr, sk, fk

    def block_product_sq(self) -> torch.Tensor:
        """g_k^2 = ||M^k N_k||_F^2 for every block (segmented square sums: int8
        tensor-core Ozaki split, or DMMA; see segsq_engine)."""
        eng = segsq_engine(self.max_len, self.M.shape[0], self.N.shape[1], self.n)
        if eng == "gram":
            return segsq_gram(self.M, self.N, self.offsets, self.K)
        if eng == "i8":
            return segsq_i8(self.M, self.N, self.offsets, self.K)
        return segsq(self.M, self.N, self.offsets, self.K)


SEGSQ_I8_MAX_LEN = 32768  # bmm_segsq_i8's exact-accumulation bound per segment
SEGSQ_I8_MIN_FLOPS = 2e9  # below this the DMMA kernel's single pass beats split + int8 contraction
SEGSQ_GRAM_MAX_LEN = 64   # bmm_segsq_gram: one 64 x 64 Gram panel per block
SEGSQ_I8_SPEEDUP = 3.0    # int8 Ozaki contraction vs DMMA per float64 flop (measured)


def segsq_engine(max_len: int, m: int, p: int, n: int) -> str:
    """Kernel for the OPL block-product norms g_k^2 (plan.py:176-189).

    "gram" (bmm_segsq_gram: <M^k^T M^k, N_k N_k^T> on DMMA, 36 of 64 tiles by
    symmetry, 2 (m+p) n L (36/64) flops) when every block has at most 64
    columns and that beats the direct product; else "i8" (bmm_segsq_i8, int8
    tensor cores, float64-accurate Ozaki split) for 2 m p n >= SEGSQ_I8_MIN_FLOPS
    unless a block exceeds its length bound; else "dmma" (bmm_segsq_f64, the
    direct segmented product).  BMM_SEGSQ=gram|i8|dmma forces one where it applies."""
    forced = os.environ.get("BMM_SEGSQ", "").lower()
    gram_ok = max_len <= SEGSQ_GRAM_MAX_LEN
    i8_ok = max_len <= SEGSQ_I8_MAX_LEN
    if forced == "gram" and gram_ok:
        return "gram"
    if forced in ("dmma", "f64"):
        return "dmma"
    if forced == "i8" and i8_ok:
        return "i8"
    direct = "i8" if i8_ok and 2.0 * m * p * n >= SEGSQ_I8_MIN_FLOPS else "dmma"
    direct_cost = m * p / (SEGSQ_I8_SPEEDUP if direct == "i8" else 1.0)
    if not forced and gram_ok and (m + p) * max_len * 36.0 / 64.0 < direct_cost:
        return "gram"
    return direct


PILOT_GRAM_MAX = 16  # two-step pilot norms by Gram matrices up to this many draws per block
GEMM_I8_MIN_FLOPS = 1e10  # below this the DMMA GEMM's single pass beats the split + int8 contraction


def gemm_engine(m: int, p: int, k: int) -> str:
    """Kernel for the float64 sampled contraction C @ D: "i8" (bmm_gemm_i8_gather,
    int8 tensor cores on Ozaki digit planes, gather fused into the split) for
    2 m p k >= GEMM_I8_MIN_FLOPS, else "dmma"; BMM_GEMM=i8|dmma forces one."""
    forced = os.environ.get("BMM_GEMM", "").lower()
    if forced in ("i8", "dmma"):
        return forced
    return "i8" if 2.0 * m * p * k >= GEMM_I8_MIN_FLOPS else "dmma"


def f32_fused(m: int, p: int) -> bool:
    """float32 compressed sketches: gather inside the tcgen05 contraction
    (bmm_gemm_f32split_gather) when the output is one 128 x 128 tile.  Each CTA
    re-gathers its A rows per column tile and its B rows per row tile, so wider
    outputs keep the separate split gather (measured, tools/fused_probe.py,
    4096 x 1024 sketches of 680 distinct columns: 128 x 128 outputs 1.34 ms
    fused vs 1.76 ms for 2048 problems; 256 x 256 outputs 1.27 vs 0.96 ms for
    512 problems); BMM_F32_FUSED=0|1 forces either."""
    forced = os.environ.get("BMM_F32_FUSED", "")
    if forced in ("0", "1"):
        return forced == "1"
    return m <= 128 and p <= 128


def f16_fused(m: int, p: int, W: int) -> bool:
    """float32 compressed sketches with outputs of at most one 256 x 256 tile
    (config 5): gather, fp16 split and contraction in one kernel
    (bmm_gemm_f16split_gather: every sketch element gathered once, no split
    operands in HBM).  Its accumulator is not promoted, so only for W <= 1024
    (error <= ~5e-6).  Single 128 x 128 tiles keep bmm_gemm_f32split_gather;
    BMM_F16_FUSED=0|1 forces the choice."""
    forced = os.environ.get("BMM_F16_FUSED", "")
    if forced in ("0", "1"):
        return forced == "1" and W <= 1024
    return m <= 256 and p <= 256 and not (m <= 128 and p <= 128) and W <= 1024


def segsq(A: torch.Tensor, B: torch.Tensor, seg: torch.Tensor, nseg: int) -> torch.Tensor:
    if A.dtype != torch.float64:
        A = A.to(torch.float64)
    if B.dtype != torch.float64:
        B = B.to(torch.float64)
    m, p = A.shape[0], B.shape[1]
    out = torch.empty(nseg, dtype=torch.float64, device=A.device)
    wsb = _lib.load().bmm_segsq_f64_workspace(m, p, nseg, 1)
    ws = _lib.workspace(wsb)
    _lib.call("bmm_segsq_f64", _lib.ptr(A), A.stride(0), 0, _lib.ptr(B), B.stride(0), 0, m, p,
              _lib.ptr(seg), nseg, 0, 1, _lib.ptr(out), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    return out


def segsq_gram(A: torch.Tensor, B: torch.Tensor, seg: torch.Tensor, nseg: int) -> torch.Tensor:
    """g_j^2 = ||A[:, seg_j] B[seg_j, :]||_F^2 through the Gram identity on the
    DMMA pipe (bmm_segsq_gram; segments of at most 64 columns)."""
    if A.dtype != B.dtype:
        A, B = A.to(torch.float64), B.to(torch.float64)
    m, p = A.shape[0], B.shape[1]
    out = torch.empty(nseg, dtype=torch.float64, device=A.device)
    _lib.call("bmm_segsq_gram", _lib.matrix_dtype(A), _lib.ptr(A), A.stride(0), 0, _lib.ptr(B), B.stride(0), 0,
              m, p, _lib.ptr(seg), nseg, 0, 1, _lib.ptr(out), _lib.stream_ptr())
    return out


def segsq_i8(A: torch.Tensor, B: torch.Tensor, seg: torch.Tensor, nseg: int, n_inner: int | None = None
             ) -> torch.Tensor:
    """g_j^2 = ||A[:, seg_j] B[seg_j, :]||_F^2 on the int8 tensor cores (Ozaki
    split, float64 accuracy; bmm_segsq_i8).  float32 or float64 operands."""
    if A.dtype != B.dtype or A.dtype not in (torch.float32, torch.float64):
        raise TypeError("segsq_i8: A and B must both be float32 or float64")
    A, B = A.contiguous(), B.contiguous()
    m, p = A.shape[0], B.shape[1]
    n_inner = A.shape[1] if n_inner is None else n_inner
    out = torch.empty(nseg, dtype=torch.float64, device=A.device)
    ws = _lib.workspace(_lib.load().bmm_segsq_i8_workspace(m, p, n_inner, nseg, 1))
    _lib.call("bmm_segsq_i8", _lib.matrix_dtype(A), _lib.ptr(A), A.stride(0), 0, _lib.ptr(B), B.stride(0), 0,
              m, p, n_inner, _lib.ptr(seg), nseg, 0, 1, _lib.ptr(out), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    return out


def split_blocks(flat: np.ndarray, part: BlockPartition) -> tuple:
    off = part.offsets
    return tuple(flat[off[k]:off[k + 1]].copy() for k in range(part.num_blocks))


def raise_status(st: int, diag: int, c: int) -> None:
    """Map a device status code to the reference's exception."""
    if st == _lib.ST_OK:
        return
    msgs = {
        _lib.ST_ZERO_SCORE: "all blocks have zero score: nothing to sample",
        _lib.ST_CAUCHY_SCHWARZ: "exact product norm exceeds score sum (Cauchy-Schwarz violated)",
        _lib.ST_RADICAND: "radicand negative beyond rounding slack",
        _lib.ST_ALL_ZERO_WEIGHT: "all weights are zero",
        _lib.ST_BAD_WEIGHT: "weights must be finite and >= 0",
        _lib.ST_CAP_BELOW_FLOOR: "some cap lies below the required floor of 1",
        _lib.ST_BELOW_FLOORS: f"budget c={c} is below the {diag} required floors",
        _lib.ST_ABOVE_CAPS: f"budget c={c} exceeds the total caps {diag}",
        _lib.ST_EMPTY_SUPPORT: "probability vector has empty support",
        _lib.ST_PLAN_MISMATCH: f"block {diag}: zero budget and zero-probability flag must coincide",
        _lib.ST_BAD_PROBS: f"block {diag}: probabilities must be finite and >= 0",
    }
    if st == _lib.ST_NO_CONVERGE:
        raise AssertionError("apportionment did not converge")
    if st == _lib.ST_NOT_PLACED:
        raise AssertionError("apportionment failed to place the full budget")
    raise ValueError(msgs.get(st, f"device status {st}"))


def device_budgets(rule: int, K: int, c: int, *, s=None, aux=None, sizes=None, caps=None,
                   floors=None, cap=True):
    """Run bmm_budgets for one problem; returns (budgets int64 ndarray, notes flag)."""
    dev = _lib.device()
    budgets = torch.empty(K, dtype=torch.int64, device=dev)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    diag = torch.empty(1, dtype=torch.int64, device=dev)
    notes = torch.empty(1, dtype=torch.int32, device=dev)
    ws = _lib.workspace(_lib.load().bmm_budgets_workspace(K))
    cd = _lib.i64([c])
    _lib.call("bmm_budgets", rule, _lib.ptr(s), _lib.ptr(aux), _lib.ptr(sizes), _lib.ptr(caps),
              _lib.ptr(floors), K, 1, _lib.ptr(cd), int(bool(cap)), _lib.ptr(budgets), None,
              _lib.ptr(status), _lib.ptr(diag), _lib.ptr(notes), _lib.ptr(ws), _lib.stream_ptr())
    st, dg, nt = int(status.item()), int(diag.item()), int(notes.item())
    raise_status(st, dg, c)
    return _lib.host(budgets), nt


# ---------------------------------------------------------------- public API

def score_sums(M, N, part: BlockPartition):
    """s_k = sum over block k of ||M col|| * ||N row|| (plan.py:170-173)."""
    inst = DeviceInstance(M, N, part)
    _, s, _ = inst.block_stats(probs=False, s=True)
    return _lib.host(s) if _lib.want_numpy(M, N) else s


def block_scores(M, N, part: BlockPartition) -> BlockScores:
    """Score sums and exact block-product norms (plan.py:176-189)."""
    inst = DeviceInstance(M, N, part)
    _, s, _ = inst.block_stats(probs=False, s=True)
    g = torch.sqrt(inst.block_product_sq())
    return BlockScores(_lib.host(s), _lib.host(g), exact=True)


def optimal_probabilities(M, N, part: BlockPartition) -> BlockProbabilities:
    """p_i proportional to ||M col i|| * ||N row i|| per block (plan.py:192-206)."""
    inst = DeviceInstance(M, N, part)
    pr, _, _ = inst.block_stats(probs=True, s=False)
    return BlockProbabilities(split_blocks(_lib.host(pr), part), rule="optimal")


def uniform_probabilities(part: BlockPartition) -> BlockProbabilities:
    """1/n_k within every block (plan.py:209-212)."""
    return BlockProbabilities(tuple(np.full(nk, 1.0 / nk) for nk in part.sizes), rule="uniform")


def integerize(weights, c: int, caps=None, floor=None) -> np.ndarray:
    """Largest-remainder split of c into integer block counts with floors and
    caps (plan.py:242-347), on device (bmm_budgets, rule EXPLICIT)."""
    w = np.asarray(weights, dtype=np.float64)
    if w.ndim != 1 or w.size == 0:
        raise ValueError("weights must be a nonempty vector")
    if not np.isfinite(w).all() or (w < 0).any():
        raise ValueError("weights must be finite and >= 0")
    if not (w > 0).any():
        raise ValueError("all weights are zero")
    c = int(c)
    if c < 0:
        raise ValueError("budget must be >= 0")
    K = w.size
    fl = None
    if floor is not None:
        fl = np.asarray(floor, dtype=bool)
        if fl.shape != (K,):
            raise ValueError("floor mask must have one entry per block")
    cp = None
    if caps is not None:
        cp = np.asarray(caps, dtype=np.int64)
        if cp.shape != (K,):
            raise ValueError("caps must have one entry per block")
    dev = _lib.device()
    wd = _lib.f64(w)
    capd = _lib.i64(cp) if cp is not None else None
    fld = torch.as_tensor(fl.astype(np.uint8), device=dev) if fl is not None else None
    budgets, _ = device_budgets(_lib.RULE_EXPLICIT, K, c, aux=wd, caps=capd, floors=fld)
    return budgets


def optimal_size_weights(M, N, part: BlockPartition) -> np.ndarray:
    """sqrt(s_k^2 - g_k^2) with exact g_k (plan.py:350-361)."""
    sc = block_scores(M, N, part)
    # K-length bookkeeping on the device-computed s and g
    rad = sc.score_sums ** 2 - sc.product_norms ** 2
    bad = rad < -RADICAND_SLACK * sc.score_sums ** 2
    if bad.any():
        raise ValueError(f"radicand negative beyond rounding slack in blocks {np.where(bad)[0]}")
    return np.sqrt(np.maximum(rad, 0.0))


def real_optimal_budgets(M, N, part: BlockPartition, c: int) -> np.ndarray:
    """c * w_k / sum(w) before integerization (plan.py:364-370)."""
    w = optimal_size_weights(M, N, part)
    tot = w.sum()
    if tot == 0.0:
        raise ValueError("all optimal size weights are zero")
    return c * w / tot


_FALLBACK_NOTES = {
    "OPL": ("optimal size weights all zero; fell back to score-sum sizes",),
    "TWO": ("pilot size weights all zero; fell back to score-sum sizes",),
}


def allocate_optimal(M, N, part: BlockPartition, c: int, cap: bool = True) -> SamplingPlan:
    """Variance-minimising plan, tag OPL (plan.py:383-400; Eq. 3.9)."""
    inst = DeviceInstance(M, N, part)
    pr, s, _ = inst.block_stats(probs=True, s=True)
    gsq = inst.block_product_sq()
    budgets, note = device_budgets(_lib.RULE_OPL, inst.K, int(c), s=s, aux=gsq, sizes=inst.sizes, cap=cap)
    probs = BlockProbabilities(split_blocks(_lib.host(pr), part), rule="optimal")
    return SamplingPlan(part, probs, budgets, method="OPL", notes=_FALLBACK_NOTES["OPL"] if note else ())


def allocate_by_score_sums(M, N, part: BlockPartition, c: int, cap: bool = True) -> SamplingPlan:
    """Score-sum sizes, tag ONC (plan.py:403-413; Eq. 4.2)."""
    inst = DeviceInstance(M, N, part)
    pr, s, _ = inst.block_stats(probs=True, s=True)
    budgets, _ = device_budgets(_lib.RULE_ONC, inst.K, int(c), s=s, sizes=inst.sizes, cap=cap)
    probs = BlockProbabilities(split_blocks(_lib.host(pr), part), rule="optimal")
    return SamplingPlan(part, probs, budgets, method="ONC")


def allocate_uniform(part: BlockPartition, c: int, cap: bool = True) -> SamplingPlan:
    """Uniform probabilities and c/K sizes, tag UU (plan.py:416-421)."""
    budgets, _ = device_budgets(_lib.RULE_UU, part.num_blocks, int(c), sizes=_lib.i64(part.sizes), cap=cap)
    return SamplingPlan(part, uniform_probabilities(part), budgets, method="UU")


def allocate_two_step(M, N, part: BlockPartition, c: int, c0: int, p0: BlockProbabilities,
                      rng: np.random.Generator, cap: bool = True,
                      method: Optional[str] = None) -> SamplingPlan:
    """Pilot-then-allocate plan, tags ONU/ONMCNR (plan.py:424-480; Alg. 3).

    floor(c0/K) pilot draws per block on child streams rng.spawn(K); the pilot
    norms ||C0 D0||_F come from the DMMA segmented square-sum GEMM."""
    from .estimators import sample_blocks  # estimators builds on plans

    _check_instance(M, N, part)
    p0.check_partition(part)
    K = part.num_blocks
    pilot_count = int(c0) // K
    if pilot_count < 1:
        raise ValueError(f"c0={c0} gives no pilot draws for K={K} blocks")
    inst = DeviceInstance(M, N, part)
    _, s, _ = inst.block_stats(probs=False, s=True)
    s_host = _lib.host(s)
    if s_host.sum() == 0.0:
        raise ValueError("all blocks have zero score: nothing to sample")
    live = np.array([v.sum() != 0.0 for v in p0.per_block])
    for k in np.flatnonzero(live):  # sketch_columns validation (estimators.py:75-76)
        if abs(p0[k].sum() - 1.0) > 1e-9:
            raise ValueError("probabilities must be >= 0 and sum to 1")
    words, first = _rng.spawn_words(rng, K)
    pilot_budgets = np.where(live, pilot_count, 0).astype(np.int64)
    col, prob, scale, col_off = sample_blocks(inst, p0.flat(), pilot_budgets, words, first)
    W0 = int(col_off[-1].item()) if K else 0
    if W0 > 0:
        # ||C0_k D0_k||_F^2 with the pilot sketch gathered on the fly (plan.py:463-464)
        m, p = inst.M.shape[0], inst.N.shape[1]
        pilot_sq = torch.empty(K, dtype=torch.float64, device=inst.M.device)
        if int(pilot_budgets.max()) <= PILOT_GRAM_MAX:  # few draws per block: Gram matrices
            _lib.call("bmm_segsq_gram_gather", _lib.matrix_dtype(inst.M), _lib.ptr(inst.M), inst.M.stride(0), 0,
                      _lib.ptr(inst.N), inst.N.stride(0), 0, m, p, _lib.ptr(col), _lib.ptr(scale), W0,
                      _lib.ptr(col_off), K, 0, int(pilot_budgets.max()), 1, _lib.ptr(pilot_sq), _lib.stream_ptr())
        else:
            A = inst.M if inst.M.dtype == torch.float64 else inst.M.to(torch.float64)
            B = inst.N if inst.N.dtype == torch.float64 else inst.N.to(torch.float64)
            ws = _lib.workspace(_lib.load().bmm_segsq_f64_workspace(m, p, K, 1))
            _lib.call("bmm_segsq_f64_gather", _lib.ptr(A), A.stride(0), 0, _lib.ptr(B), B.stride(0), 0, m, p,
                      _lib.ptr(col), _lib.ptr(scale), W0, _lib.ptr(col_off), K, 0, 1, _lib.ptr(pilot_sq),
                      _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    else:
        pilot_sq = torch.zeros(K, dtype=torch.float64, device=s.device)
    budgets, note = device_budgets(_lib.RULE_TWO_STEP, K, int(c), s=s, aux=pilot_sq, sizes=inst.sizes,
                                   cap=cap)
    pilot = torch.sqrt(pilot_sq)
    if method is None:
        method = "ONU" if p0.rule == "uniform" else "ONMCNR"
    pr, _, _ = inst.block_stats(probs=True, s=False)
    probs = BlockProbabilities(split_blocks(_lib.host(pr), part), rule="optimal")
    return SamplingPlan(part, probs, budgets, method=method,
                        notes=_FALLBACK_NOTES["TWO"] if note else (), pilot_norms=_lib.host(pilot))


def block_norm_probabilities(M, N, part: BlockPartition):
    """Whole-block probabilities q_k ∝ ||M^k||_F ||N_k||_F, tag SSM (plan.py:483-496)."""
    inst = DeviceInstance(M, N, part)
    q, st = inst_block_q(inst)
    if st != _lib.ST_OK:
        raise ValueError("all blocks have zero norm: nothing to sample")
    return _lib.host(q) if _lib.want_numpy(M, N) else q


def inst_block_q(inst: DeviceInstance):
    _, _, f = inst.block_stats(probs=False, s=False, fnorm=True)
    q = torch.empty(inst.K, dtype=torch.float64, device=f.device)
    status = torch.empty(1, dtype=torch.int32, device=f.device)
    _lib.call("bmm_normalize", _lib.ptr(f), inst.K, 1, _lib.ptr(q), _lib.ptr(status), _lib.stream_ptr())
    return q, int(status.item())


# ---------------------------------------------------------------- plan documents

class FloorRatio(NamedTuple):
    """plan.py:215-217."""

    ratio: float
    support_mismatch: bool


def prob_floor_ratio(probs: BlockProbabilities, reference: BlockProbabilities) -> FloorRatio:
    """Largest beta with probs >= beta * reference on reference's support,
    clamped to [0, 1]; (0, True) when probs vanishes there (plan.py:220-239)."""
    if len(probs.per_block) != len(reference.per_block):
        raise ValueError("block counts differ")
    ratio = 1.0
    for p, r in zip(probs.per_block, reference.per_block):
        p, r = np.asarray(p), np.asarray(r)
        if p.shape != r.shape:
            raise ValueError("per-block shapes differ")
        sup = r > 0
        if not sup.any():
            continue
        if (p[sup] == 0).any():
            return FloorRatio(0.0, True)
        ratio = min(ratio, float((p[sup] / r[sup]).min()))
    return FloorRatio(min(max(ratio, 0.0), 1.0), False)


def plan_to_dict(plan: SamplingPlan, include_probs: Optional[bool] = None) -> dict:
    """JSON document of a plan (plan.py:499-518): probabilities are written
    only when no named rule regenerates them, unless forced."""
    if plan.method not in METHOD_TAGS:
        raise ValueError(f"method tag {plan.method!r} not in {METHOD_TAGS}")
    if include_probs is None:
        include_probs = plan.probs.rule == "explicit"
    doc = {"method": plan.method, "partition": list(plan.partition.sizes), "total": plan.total,
           "budgets": [int(b) for b in plan.budgets], "probs_rule": plan.probs.rule}
    if include_probs:
        doc["probs"] = [np.asarray(p).tolist() for p in plan.probs.per_block]
    if plan.pilot_norms is not None:
        doc["pilot_norms"] = np.asarray(plan.pilot_norms).tolist()
    return doc


def plan_from_dict(doc: dict, M=None, N=None) -> SamplingPlan:
    """plan.py:521-549; 'optimal' probabilities are regenerated on device from M, N."""
    part = BlockPartition(tuple(doc["partition"]))
    rule = doc.get("probs_rule", "explicit")
    if "probs" in doc:
        probs = BlockProbabilities(tuple(np.asarray(p) for p in doc["probs"]), rule=rule)
    elif rule == "uniform":
        probs = uniform_probabilities(part)
    elif rule == "optimal":
        if M is None or N is None:
            raise ValueError("regenerating 'optimal' probabilities requires the factor matrices")
        probs = optimal_probabilities(M, N, part)
    else:
        raise ValueError(f"cannot reconstruct probabilities for rule {rule!r}")
    pilot = doc.get("pilot_norms")
    plan = SamplingPlan(part, probs, np.asarray(doc["budgets"], dtype=np.int64), method=doc.get("method", ""),
                        pilot_norms=None if pilot is None else np.asarray(pilot))
    if plan.total != doc.get("total", plan.total):
        raise ValueError("budget sum disagrees with the recorded total")
    return plan


def plan_to_json(plan: SamplingPlan, include_probs: Optional[bool] = None) -> str:
    return json.dumps(plan_to_dict(plan, include_probs), indent=2)


def plan_from_json(text: str, M=None, N=None) -> SamplingPlan:
    return plan_from_dict(json.loads(text), M, N)
