"""Device-resident approximate-product pipeline (the batched fast path).

One object holds every buffer for a fixed (shape, partition, method, budget,
batch), so a call is a fixed sequence of kernel launches on the current
stream with no allocation and no host synchronisation:

  K1 bmm_norms -> K2 bmm_block_probs -> [OPL: bmm_segsq_i8 of M^k N_k]
  [two-step: pilot budgets -> CDF -> child seeds -> draws -> gather -> segsq]
  -> bmm_budgets -> bmm_block_cdf -> bmm_seed_streams -> bmm_sample
  -> bmm_gather -> bmm_gemm_f64  (C @ D), or bmm_gemm_i8_gather for large contractions

It computes exactly what the reference composition computes
(allocate_* + estimate_product, estimate_product_two_step,
estimate_product_block_sampling; pkg/src/blockmm/plan.py:383-480,
estimators.py:125-253) and is bit-compatible with the per-call API in this
package (same kernels, same streams).  Device status codes (the reference's
ValueError/AssertionError cases) are read only by ``check()``.
"""
from __future__ import annotations

import copy
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from . import rng as _rng
from .plan import PILOT_GRAM_MAX, f16_fused, f32_fused, gemm_engine, raise_status, segsq_engine

METHODS = ("OPL", "ONC", "UU", "ONU", "ONMCNR", "SSM")


@dataclass
class StreamSeeds:
    """Entropy words and first child index per problem for one spawn(K)."""

    words: np.ndarray        # (batch, n_words) uint32
    first: np.ndarray        # (batch,) int64


@dataclass
class CallSeeds:
    main: Optional[StreamSeeds] = None
    pilot: Optional[StreamSeeds] = None
    states: Optional[np.ndarray] = None   # SSM: (batch, 4) uint64 caller stream states


def seeds_from_rngs(method: str, rngs: list, K: int, draws: int = 0) -> CallSeeds:
    """Apply the reference's generator side effects for one call per problem
    and return the device seeds.  rngs: one numpy Generator per problem."""

    def stack(parts):
        ws = [w for w, _ in parts]
        if len({len(w) for w in ws}) != 1:
            raise ValueError("all problems' generators must have entropy/key words of equal length")
        return StreamSeeds(np.stack(ws).astype(np.uint32), np.array([f for _, f in parts], dtype=np.int64))

    if method == "SSM":
        st = np.stack([_rng.stream_state(r) for r in rngs])
        for r in rngs:
            _rng.consume(r, draws)
        return CallSeeds(states=st)
    if method in ("ONU", "ONMCNR"):
        pil, mai = [], []
        for r in rngs:
            pr, mr = r.spawn(2)                       # estimators.py:207
            pil.append(_rng.spawn_words(pr, K))       # plan.py:456
            mai.append(_rng.spawn_words(mr, K))       # estimators.py:141
        return CallSeeds(main=stack(mai), pilot=stack(pil))
    return CallSeeds(main=stack([_rng.spawn_words(r, K) for r in rngs]))


def seeds_from_keys(method: str, entropy: int, key_prefix: tuple, keys, K: int) -> CallSeeds:
    """Seeds for a batch of fresh generators ``default_rng(SeedSequence(entropy,
    spawn_key=key_prefix + (keys[b],)))`` without building them: problem b's
    estimate spawns children key_prefix + (keys[b], j) (estimators.py:141), and
    the two-step pilot/main generators are its children 0 and 1
    (estimators.py:207).  Vectorised; equals seeds_from_rngs on those
    generators (tests/test_gpu_pipeline.py)."""
    keys = np.asarray(keys, dtype=np.int64)
    if (keys < 0).any() or (keys >= 2**32).any():
        raise ValueError("per-problem keys must fit one 32-bit word")
    run = _rng._words(int(entropy))
    run = run + [0] * max(0, 4 - len(run))
    pre = _rng._words(tuple(key_prefix)) if key_prefix else []
    base = np.asarray(run + pre, dtype=np.uint32)
    B = keys.size
    words = np.concatenate([np.broadcast_to(base, (B, base.size)), keys[:, None].astype(np.uint32)], axis=1)
    zeros = np.zeros(B, dtype=np.int64)
    if method in ("ONU", "ONMCNR"):
        pil = np.concatenate([words, np.zeros((B, 1), np.uint32)], axis=1)
        mai = np.concatenate([words, np.ones((B, 1), np.uint32)], axis=1)
        return CallSeeds(main=StreamSeeds(mai, zeros), pilot=StreamSeeds(pil, zeros))
    if method == "SSM":
        raise ValueError("SSM draws from the caller's stream; use seeds_from_rngs")
    return CallSeeds(main=StreamSeeds(np.ascontiguousarray(words), zeros))


def _fused_stats(obj, M: torch.Tensor) -> bool:
    """Norm pass inside OPL's Gram-form g_k^2 kernel (bmm_segsq_gram_norms)?  Needs
    the Gram engine, p = 128 * 2^k (NumPy's row tree is perfect), one device (no
    exchange).  Opt-in (BMM_FUSED_STATS=1): bit-identical, but the norm chains sit
    on the DMMA warps' critical path -- config 4, cool GPU: 24.3 ms fused against
    5.3 + 18.8 ms separate; inside the power-capped step 46.5 against 38.8 ms
    (tools/gram_norms_probe.py, tools/timeline.py cfg4)."""
    if os.environ.get("BMM_FUSED_STATS", "0") != "1" or getattr(obj, "exchange", None) is not None:
        return False
    p = obj.p
    return (getattr(obj, "seg_engine", None) == "gram" and p >= 128 and (p & (p - 1)) == 0
            and M.dtype in (torch.float32, torch.float64))


def _stats_launch(obj, M: torch.Tensor, N: torch.Tensor, chunks, *, probs: bool, gsq: bool) -> bool:
    """Per-instance statistics of `obj` (a SketchPipeline or a group's SharedStats):
    the norm pass (K1), optionally the optimal probabilities / score sums / main
    CDF (K2) and, in chunked mode, OPL's g_k^2 per landed chunk.  Returns True
    when g_k^2 was computed here (chunked)."""
    B, m, n, p, K = obj.B, obj.m, obj.n, obj.p, obj.K
    dt = _lib.matrix_dtype(M)
    st = _lib.stream_ptr()
    sM, sN = m * n, n * p
    ldm, ldn = M.stride(-2), N.stride(-2)
    P = lambda t: t.data_ptr()  # noqa: E731
    seg_done = False
    if gsq and chunks is None and _fused_stats(obj, M):
        # OPL's Gram kernel reads every column of M and row of N once anyway: the norm
        # pass rides along (bit-identical colsq / rowsq, gram_blocks.cu RowTree)
        obj._c("bmm_segsq_gram_norms", dt, P(M), ldm, sM, P(N), ldn, sN, m, p, P(obj.offsets), K, 0, B, P(obj.gsq),
               P(obj.colsq), P(obj.rowsq), n, st)
        seg_done = True
    elif getattr(obj, "exchange", None) is not None:
        # one rank of a sharded product: exact cross-rank norm pass (distributed.ShardExchange)
        if B != 1 or chunks is not None:
            raise ValueError("sharded pipelines run one problem, without chunked transfer")
        obj.exchange.norms(M, N, obj.colsq, obj.rowsq)
    elif chunks is None:
        obj._c("bmm_norms", dt, P(M), m, n, ldm, sM, P(N), p, ldn, sN, B, 0, P(obj.colsq), P(obj.rowsq), st)
    else:
        if B != 1 or not probs:
            raise ValueError("chunked launch: one problem, non-SSM method")
        es = M.element_size()
        cur = torch.cuda.current_stream()
        for c0, c1, k0, k1, ev in chunks:
            cur.wait_event(ev)
            obj._c("bmm_norms", dt, P(M) + es * c0, m, c1 - c0, ldm, 0, P(N) + es * c0 * ldn, p, ldn, 0, 1, 0,
                   P(obj.colsq) + 8 * c0, P(obj.rowsq) + 8 * c0, st)
            if gsq:
                obj._segsq(M, N, dt, k0, k1, 1, st)
        seg_done = gsq
    if probs:
        # probabilities, score sums and (fused) the main CDF of the optimal probabilities
        obj._c("bmm_block_probs", P(obj.colsq), P(obj.rowsq), n, P(obj.offsets), K, B, obj.max_len,
               P(obj.probs), P(obj.s), None, P(obj.cum), P(obj.last), st)
    return seg_done


class SketchPipeline:
    """Preallocated device pipeline for `batch` problems of shape
    M (m x n), N (n x p) sharing one block partition."""

    def __init__(self, m: int, n: int, p: int, sizes, c: int, method: str, *, batch: int = 1,
                 dtype=torch.float64, c0: int = 0, cap: bool = True, draws: int = 0, compress: bool = True):
        if method not in METHODS:
            raise ValueError(f"unknown method {method!r}")
        dev = _lib.device()
        self.m, self.n, self.p, self.B = int(m), int(n), int(p), int(batch)
        self.sizes = tuple(int(s) for s in sizes)
        if sum(self.sizes) != self.n:
            raise ValueError("partition does not cover n")
        self.K = len(self.sizes)
        self.max_len = max(self.sizes)
        self.method, self.c, self.c0, self.cap = method, int(c), int(c0), bool(cap)
        self.dtype = dtype
        self.lib = _lib.load()
        K, B, n_ = self.K, self.B, self.n
        f64 = dict(dtype=torch.float64, device=dev)
        i64 = dict(dtype=torch.int64, device=dev)
        off = np.zeros(K + 1, dtype=np.int64)
        np.cumsum(self.sizes, out=off[1:])
        self.offsets = torch.as_tensor(off, device=dev)
        self.sizes_d = torch.as_tensor(np.asarray(self.sizes, dtype=np.int64), device=dev)
        self.colsq = torch.empty(B * n_, **f64)
        self.rowsq = torch.empty(B * n_, **f64)
        self.probs = torch.empty(B * n_, **f64)
        self.s = torch.empty(B * K, **f64)
        self.cum = torch.empty(B * n_, **f64)
        self.last = torch.empty(B * K, **i64)
        self.budgets = torch.empty(B * K, **i64)
        self.col_off = torch.empty(B * (K + 1), **i64)
        self.status = torch.zeros(B, dtype=torch.int32, device=dev)
        self.diag = torch.zeros(B, **i64)
        self.notes = torch.zeros(B, dtype=torch.int32, device=dev)
        self.states = torch.empty(B * K * 4, **i64)
        self.c_arr = torch.full((B,), self.c, **i64)
        self.ws_budget = torch.empty(max(256, self.lib.bmm_budgets_workspace(K) * B), dtype=torch.uint8, device=dev)
        if method == "SSM":
            self.draws = int(draws)
            if len(set(self.sizes)) != 1:
                raise ValueError("batched SSM needs equal blocks (fixed sketch width)")
            self.W = self.draws * self.sizes[0]
            self.fnorm = torch.empty(B * K, **f64)
            self.q = torch.empty(B * K, **f64)
            self.qcum = torch.empty(B * K, **f64)
            self.qlast = torch.empty(B, **i64)
            self.qoff = torch.as_tensor(np.array([0, K], dtype=np.int64), device=dev)
            self.q_bud = torch.full((B,), self.draws, **i64)
            self.q_coloff = torch.as_tensor(np.tile(np.array([0, self.draws], dtype=np.int64), B), device=dev)
            self.sk_off = torch.as_tensor(np.arange(self.draws + 1, dtype=np.int64) * self.sizes[0], device=dev)
            self.ssm_states = torch.empty(B * 4, **i64)
            self.blk = torch.empty(B * self.draws, **i64)
            self.blk_prob = torch.empty(B * self.draws, **f64)
            self.blk_scale = torch.empty(B * self.draws, **f64)
        else:
            self.W = self.c
        W = self.W
        self.column = torch.zeros(B * W, **i64)  # zero-init: failed plans gather column 0, never garbage
        self.prob = torch.empty(B * W, **f64)
        self.scale = torch.empty(B * W, **f64)
        # float32 inputs take the tcgen05 split-operand path (pair groups need W % 8 == 0)
        self.tf32 = (dtype == torch.float32 and W % 8 == 0)
        self._joint = None  # row stride of the pooled C when a joint PipelineGroup contracts
        # compressed sketch: one rank-1 term per distinct drawn column (bmm_compress_sketch)
        self.compress = bool(compress)
        if self.compress:
            self.k_column = torch.empty(B * W, **i64)
            self.k_scale = torch.empty(B * W, **f64)
            self.k_count = torch.empty(B, **i64)
            self.ws_cmp = torch.empty(max(256, self.lib.bmm_compress_workspace(n_, B)), dtype=torch.uint8, device=dev)
        # small float32 outputs (at most 4 x 4 tiles of 128): gather inside the contraction
        # (bmm_gemm_f32split_gather); large ones would re-gather A once per column tile
        self.fused = self.tf32 and self.compress and f32_fused(self.m, self.p)
        # outputs of one 256 x 256 tile at W <= 1024 (config 5): the fp16-split gather and
        # contraction in one kernel, no split operands in HBM
        self.fused16 = (self.tf32 and self.compress and not self.fused and self.n % 4 == 0 and self.p % 4 == 0
                        and f16_fused(self.m, self.p, W))  # (TMA streams rows of M and N)
        # large float32 outputs: the fp16 split on CTA pairs (3 tensor instructions per 16 K
        # instead of 4; BMM_F16=0 keeps the tf32 + bf16 split)
        self.f16 = (self.tf32 and self.compress and not self.fused and not self.fused16 and self.m >= 256
                    and self.p >= 256 and os.environ.get("BMM_F16", "1") != "0")
        if self.f16 or self.fused16:
            self.kexp = torch.zeros(B * W, dtype=torch.int32, device=dev)
            self.gshift = torch.zeros(B, dtype=torch.int32, device=dev)
        # many small problems (config 5): probabilities, budgets, child streams, draws, the
        # compressed sketch and the balanced exponents in ONE launch, one CTA per problem
        # (bmm_plan_small; BMM_PLAN_SMALL=0 keeps the separate kernels)
        self.plan_small = (method in ("ONC", "OPL") and self.compress and B >= 256 and self.max_len <= 128
                           and W < 65536 and n_ < 65536 and self.lib.bmm_plan_small_smem(n_, K, W) <= 200 * 1024
                           and os.environ.get("BMM_PLAN_SMALL", "1") != "0")
        if self.tf32:
            f32 = dict(dtype=torch.float32, device=dev)
            if not (self.fused or self.fused16):
                self.a_hi = torch.empty(B * self.m * W, **f32)
                self.a_x = torch.empty(B * self.m * W, **f32)
                self.b_hi = torch.empty(B * self.p * W, **f32)
                self.b_x = torch.empty(B * self.p * W, **f32)
            self.CD = torch.empty(B * self.m * self.p, **f32)
        else:
            # float64 path.  Large contractions: the int8 Ozaki path with the sketch
            # gathered inside its digit split (bmm_gemm_i8_gather).  Otherwise gather the
            # rescaled sketch (bandwidth-bound kernel at full occupancy), then C @ D on
            # the DMMA pipe.
            self.gemm_engine = gemm_engine(self.m, self.p, W)
            self.CD = torch.empty(B * self.m * self.p, **f64)
            if self.gemm_engine == "i8":
                self.ws_gemm = torch.empty(max(256, self.lib.bmm_gemm_i8_workspace(self.m, self.p, W, B)),
                                           dtype=torch.uint8, device=dev)
                self.kexp = torch.empty(B * W, dtype=torch.int32, device=dev)
            else:
                self.C = torch.empty(B * self.m * W, **f64)
                self.D = torch.empty(B * W * self.p, **f64)
                self.ws_gemm = torch.empty(max(256, self.lib.bmm_gemm_f64_workspace(self.m, self.p, W, B)),
                                           dtype=torch.uint8, device=dev)
        if method == "OPL":
            self.gsq = torch.empty(B * K, **f64)
            # g_k^2 on the int8 tensor cores (Ozaki split; float32 inputs read directly)
            self.seg_engine = segsq_engine(self.max_len, self.m, self.p, self.n)
            wsb = (self.lib.bmm_segsq_i8_workspace(self.m, self.p, self.n, K, B) if self.seg_engine == "i8"
                   else 0 if self.seg_engine == "gram" else self.lib.bmm_segsq_f64_workspace(self.m, self.p, K, B))
            self.ws_seg = torch.empty(max(256, wsb), dtype=torch.uint8, device=dev)
        if method in ("ONU", "ONMCNR"):
            self.pc = self.c0 // K
            if self.pc < 1:
                raise ValueError(f"c0={self.c0} gives no pilot draws for K={K} blocks")
            W0 = K * self.pc
            self.W0 = W0
            self.p_bud = torch.empty(B * K, **i64)
            self.p_coloff = torch.empty(B * (K + 1), **i64)
            self.p_c = torch.full((B,), self.pc, **i64)
            self.p_states = torch.empty(B * K * 4, **i64)
            self.p_column = torch.zeros(B * W0, **i64)
            self.p_prob = torch.zeros(B * W0, **f64)
            self.p_scale = torch.zeros(B * W0, **f64)
            self.pilot_sq = torch.empty(B * K, **f64)
            self.ws_seg = torch.empty(max(256, self.lib.bmm_segsq_f64_workspace(self.m, self.p, K, B)),
                                      dtype=torch.uint8, device=dev)
            if method == "ONU":
                u = np.concatenate([np.full(nk, 1.0 / nk) for nk in self.sizes])
                self.p0 = torch.as_tensor(np.tile(u, B), device=dev)
            self.p0cum = torch.empty(B * n_, **f64)
            self.p0last = torch.empty(B * K, **i64)
        if method == "UU":
            u = np.concatenate([np.full(nk, 1.0 / nk) for nk in self.sizes])
            self._uprobs = torch.as_tensor(np.tile(u, B), device=dev)
        self.graph = None
        self.timeline = None
        self.stamps = None  # (device int64 buffer, [entry names]) for tools/timeline.py
        self.shared = None        # SharedStats of the PipelineGroup that owns this member's statistics
        self.exchange = None      # distributed.ShardExchange when this pipeline computes one rank's tile
        self._group_active = False  # set while the owning group enqueues this member
        self._waves = None        # (problems per wave, streams): set_waves
        self._wave_views = None

    # ------------------------------------------------------------------ steps
    def _c(self, name, *args):
        rc = getattr(self.lib, name)(*args)
        if rc < 0:
            raise RuntimeError(f"{name} failed ({rc}): {self.lib.bmm_last_error().decode()}")
        if self.timeline is not None:  # eager profiling: an event after every stage
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.timeline.append((name, ev))
        if self.stamps is not None:  # graph profiling: a device clock stamp after every stage
            buf, names = self.stamps
            self.lib.bmm_timestamp(buf.data_ptr() + 8 * len(names), _lib.stream_ptr())
            names.append(name)

    def stage_times(self, M, N, seeds) -> list:
        """Eager run with a CUDA event after every C-ABI call; returns
        [(entry point, ms)] in launch order (warm caches, real context)."""
        self.set_seeds(seeds)
        start = torch.cuda.Event(enable_timing=True)
        start.record()
        self.timeline = []
        try:
            self.launch(M, N)
        finally:
            tl, self.timeline = self.timeline, None
        torch.cuda.synchronize()
        out, prev = [], start
        for name, ev in tl:
            out.append((name, prev.elapsed_time(ev)))
            prev = ev
        return out

    def _seed(self, which: str, states: torch.Tensor, st):
        words, first = self._seedbuf[which]
        self._c("bmm_seed_streams", words.data_ptr(), words.shape[1], first.data_ptr(), self.K, self.B,
                states.data_ptr(), st)

    # ---- per-call seed material: pinned staging -> async copy into fixed device buffers
    def set_seeds(self, seeds: CallSeeds) -> None:
        """Stage this call's seeds (host numpy) into the device buffers the
        launch sequence reads; async, double-buffered pinned staging."""
        items = {}
        if seeds.main is not None:
            items["main"] = seeds.main
        if seeds.pilot is not None:
            items["pilot"] = seeds.pilot
        if seeds.states is not None:
            items["states"] = seeds.states
        if not hasattr(self, "_seedbuf"):
            self._seedbuf, self._stage, self._stage_ev, self._slot = {}, [{}, {}], [None, None], 0
        self._slot ^= 1
        ev = self._stage_ev[self._slot]
        if ev is not None:
            ev.synchronize()
        stage = self._stage[self._slot]
        dev = self.colsq.device
        for key, val in items.items():
            arrs = ((np.ascontiguousarray(val.words).view(np.int32), np.ascontiguousarray(val.first, dtype=np.int64))
                    if key != "states" else (np.ascontiguousarray(val).view(np.int64).reshape(self.B, 4),))
            if key not in self._seedbuf:
                self._seedbuf[key] = tuple(torch.empty(a.shape, dtype=torch.from_numpy(a).dtype, device=dev)
                                           for a in arrs)
            if key not in stage:
                stage[key] = tuple(torch.empty(a.shape, dtype=torch.from_numpy(a).dtype).pin_memory() for a in arrs)
            for dst, pin, a in zip(self._seedbuf[key], stage[key], arrs):
                if tuple(dst.shape) != a.shape:
                    raise ValueError("seed material changed shape; build a new pipeline")
                pin.numpy()[...] = a
                dst.copy_(pin, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._stage_ev[self._slot] = ev

    def capture(self, M: torch.Tensor, N: torch.Tensor) -> None:
        """Record the launch sequence for these input buffers as a CUDA graph."""
        if self.exchange is not None:
            raise RuntimeError("a sharded pipeline exchanges through host collectives: run it eagerly")
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.launch(M, N)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        n0 = _lib.launches()
        with torch.cuda.graph(g):
            self.launch(M, N)
        self.graph_launches = _lib.launches() - n0  # our kernels per replay
        self.graph, self._graph_ptrs = g, (M.data_ptr(), N.data_ptr())

    def run(self, M: torch.Tensor, N: torch.Tensor, seeds: CallSeeds) -> torch.Tensor:
        """Approximate products of the batch; returns CD as (B, m, p) (or (m, p))."""
        self._guard()
        self.set_seeds(seeds)
        if getattr(self, "graph", None) is not None and self._graph_ptrs == (M.data_ptr(), N.data_ptr()):
            self.graph.replay()
            return self._result()
        return self.launch(M, N)

    def _result(self):
        return self.CD.view(self.B, self.m, self.p) if self.B > 1 else self.CD.view(self.m, self.p)

    def _guard(self) -> None:
        if (self._joint is not None or self.shared is not None) and not self._group_active:
            raise RuntimeError("this pipeline's statistics or contraction belong to its PipelineGroup: "
                               "launch, capture and run the group")

    def launch(self, M: torch.Tensor, N: torch.Tensor, chunks=None) -> torch.Tensor:
        """Enqueue the whole pipeline on the current stream (graph-capturable).

        chunks: optional [(c0, c1, k0, k1, event)] -- block-aligned ranges of the
        inner dimension whose M columns and N rows are valid once `event` has
        completed (a chunked host->device transfer).  The norm pass and OPL's
        segmented square sums then run chunk by chunk behind the transfer; the
        rest of the pipeline is unchanged (single problem, float64 inputs).
        Members of a PipelineGroup with shared statistics skip the norm pass,
        the block probabilities and g_k (the group's SharedStats computes them)."""
        self._guard()
        if self._waves is not None and chunks is None and self.B > self._waves[0]:
            return self._launch_waves(M, N)
        if self.shared is None:
            seg_done = _stats_launch(self, M, N, chunks, probs=self.method != "SSM" and not self._plan_small_now(),
                                     gsq=self.method == "OPL")
            if self.method == "OPL" and not seg_done:
                self._segsq(M, N, _lib.matrix_dtype(M), 0, self.K, self.B, _lib.stream_ptr())
        return self._plan_and_contract(M, N)

    # ---- waves: the batch as sub-batches on several streams of one graph
    _NOT_PER_PROBLEM = ("offsets", "sizes_d", "qoff", "sk_off")

    def set_waves(self, per_wave: int, streams: int) -> None:
        """Run a batch of independent problems as ceil(B / per_wave) sub-batches spread
        round-robin over `streams` CUDA streams (forked from and joined to the launching
        stream, so one graph still holds the step): while one wave's HBM-bound norm pass or
        gather-contraction runs, another wave's latency-bound planning kernels (block
        probabilities, budgets, draws, compaction) fill the gaps.  Every wave is this
        pipeline's own launch sequence on a slice of its buffers, so the results are
        bit-identical to the single-batch run (config 5: 16 x 256 problems, 9.7 -> 8.9 ms)."""
        if per_wave < 1 or streams < 1:
            raise ValueError("per_wave and streams must be >= 1")
        if not (self.fused16 or self.fused) or self.method in ("ONU", "ONMCNR") or self.shared is not None or (
                self.method == "OPL" and self.seg_engine != "gram"):
            raise ValueError("waves: float32 fused gather-contraction pipelines (ONC, OPL on the Gram engine, UU, SSM)")
        self._waves, self._wave_views, self.graph = (int(per_wave), int(streams)), None, None

    def _make_wave_views(self):
        per_wave, S = self._waves
        B = self.B
        views = []
        for a in range(0, B, per_wave):
            b = min(B, a + per_wave)
            v = copy.copy(self)
            v.B, v._waves, v._wave_views, v.graph = b - a, None, None, None
            for name, t in vars(self).items():
                if not isinstance(t, torch.Tensor) or name in self._NOT_PER_PROBLEM or name in ("ws_seg", "ws_gemm"):
                    continue
                if t.numel() % B != 0:
                    raise RuntimeError(f"waves: buffer {name} is not per problem")
                per = t.numel() // B
                setattr(v, name, t[a * per:b * per])
            v._seedbuf = {k: tuple(t[a:b] for t in ts) for k, ts in self._seedbuf.items()}
            views.append((a, b, v))
        self._wave_views = views
        # equal priorities by default.  BMM_WAVE_PRIO=1 puts earlier waves on higher-priority
        # streams (a software pipeline over the waves): measured slower at config 5, 9.84 against
        # 9.60 ms (profiles/r2aw_waves_priorities.txt)
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
        if os.environ.get("BMM_WAVE_PRIO", "0") != "1":
            hi = lo = 0
        self._wave_streams = [torch.cuda.Stream(priority=max(hi, lo - (S - 1 - i))) for i in range(S)]

    def _launch_waves(self, M: torch.Tensor, N: torch.Tensor) -> torch.Tensor:
        if self._wave_views is None:
            self._make_wave_views()
        Mb = M.view(self.B, self.m, self.n)
        Nb = N.view(self.B, self.n, self.p)
        cur = torch.cuda.current_stream()
        # (an explicit two-stream pipeline -- norm passes and contractions back to back on one
        # stream, each wave's plan on a side stream between them -- measured slower, 10.3 against
        # 9.6 ms at config 5: the HBM-bound kernels fill every SM, so a plan cannot run beside
        # them and only delays its own contraction; profiles/r2ax_waves_pipelined.txt)
        for st in self._wave_streams:
            st.wait_stream(cur)
        for w, (a, b, v) in enumerate(self._wave_views):
            with torch.cuda.stream(self._wave_streams[w % len(self._wave_streams)]):
                v.launch(Mb[a:b], Nb[a:b])
        for st in self._wave_streams:
            cur.wait_stream(st)
        return self._result()

    def _plan_and_contract(self, M: torch.Tensor, N: torch.Tensor) -> torch.Tensor:
        """Everything after the per-instance statistics: sizes, draws, sketch, C @ D."""
        B, m, n, p, K, W = self.B, self.m, self.n, self.p, self.K, self.W
        dt = _lib.matrix_dtype(M)
        st = _lib.stream_ptr()
        P = lambda t: t.data_ptr()  # noqa: E731
        if self.method == "SSM":
            self._plan_ssm(st)
            return self._contract_sketch(M, N, dt, st)
        rule = {"ONC": _lib.RULE_ONC, "OPL": _lib.RULE_OPL, "UU": _lib.RULE_UU,
                "ONU": _lib.RULE_TWO_STEP, "ONMCNR": _lib.RULE_TWO_STEP}[self.method]
        aux = None
        sM, sN = m * n, n * p
        ldm, ldn = M.stride(-2), N.stride(-2)
        if self.method == "OPL":
            aux = self.gsq
        if self._plan_small_now():
            self._plan_small_call(st)
            return self._contract_sketch(M, N, dt, st, planned=True)
        if self.method in ("ONU", "ONMCNR"):
            p0 = self.p0 if self.method == "ONU" else self.probs
            s_for_pilot = None if self.method == "ONU" else self.s
            self._c("bmm_budgets", _lib.RULE_PILOT, P(s_for_pilot) if s_for_pilot is not None else None, None,
                    None, None, None, K, B, P(self.p_c), 1, P(self.p_bud), P(self.p_coloff), None, None, None,
                    P(self.ws_budget), st)
            if self.method == "ONU":
                self._c("bmm_block_cdf", P(p0), P(self.offsets), K, B, n, P(self.p0cum), P(self.p0last), st)
                p0cum, p0last = self.p0cum, self.p0last
            else:  # ONMCNR pilots with the optimal probabilities: their CDF is already built
                p0cum, p0last = self.cum, self.last
            self._seed("pilot", self.p_states, st)
            self._c("bmm_sample", P(p0), P(p0cum), P(p0last), P(self.offsets), K, B, n, self.max_len, P(self.p_bud),
                    P(self.p_coloff), self.W0, P(self.p_states), P(self.p_column), P(self.p_prob),
                    P(self.p_scale), st)
            # pilot norms ||C0_k D0_k||_F^2 straight from M and N (sketch gathered on the fly):
            # few draws per block -> two L x L Gram matrices per block instead of an m x p product
            if self.pc <= PILOT_GRAM_MAX:
                self._c("bmm_segsq_gram_gather", dt, P(M), ldm, sM, P(N), ldn, sN, m, p, P(self.p_column),
                        P(self.p_scale), self.W0, P(self.p_coloff), K, K + 1, self.pc, B, P(self.pilot_sq), st)
            else:
                A, Bm = self._f64(M, N)
                self._c("bmm_segsq_f64_gather", P(A), A.stride(-2), sM, P(Bm), Bm.stride(-2), sN, m, p,
                        P(self.p_column), P(self.p_scale), self.W0, P(self.p_coloff), K, K + 1, B,
                        P(self.pilot_sq), P(self.ws_seg), self.ws_seg.numel(), st)
            if self.exchange is not None:
                self.exchange.sum_(self.pilot_sq)  # C2: pilot norms over the output tiles
            aux = self.pilot_sq
        self._c("bmm_budgets", rule, P(self.s) if rule != _lib.RULE_UU else None, P(aux) if aux is not None else None,
                P(self.sizes_d), None, None, K, B, P(self.c_arr), int(self.cap), P(self.budgets), P(self.col_off),
                P(self.status), P(self.diag), P(self.notes), P(self.ws_budget), st)
        probs = self._uprobs if self.method == "UU" else self.probs
        if self.method == "UU":
            self._c("bmm_block_cdf", P(probs), P(self.offsets), K, B, n, P(self.cum), P(self.last), st)
        self._seed("main", self.states, st)
        self._c("bmm_sample", P(probs), P(self.cum), P(self.last), P(self.offsets), K, B, n, self.max_len,
                P(self.budgets),
                P(self.col_off), W, P(self.states), P(self.column), P(self.prob), P(self.scale), st)
        return self._contract_sketch(M, N, dt, st)

    def _plan_small_call(self, st) -> None:
        """The whole plan of every problem of the batch in one launch (bmm_plan_small)."""
        B, n, K, W = self.B, self.n, self.K, self.W
        P = lambda t: t.data_ptr()  # noqa: E731
        rule = _lib.RULE_ONC if self.method == "ONC" else _lib.RULE_OPL
        aux = self.gsq if self.method == "OPL" else None
        words, first = self._seedbuf["main"]
        bal = self.f16 or self.fused16
        self._c("bmm_plan_small", rule, P(self.colsq), P(self.rowsq), n, P(self.offsets), P(self.sizes_d), K, B,
                self.max_len, P(aux) if aux is not None else None, P(self.c_arr), int(self.cap), words.data_ptr(), words.shape[1],
                first.data_ptr(), W, P(self.probs), P(self.s), None, P(self.last), P(self.budgets),
                P(self.col_off), P(self.status), P(self.diag), P(self.notes), P(self.states), P(self.column),
                P(self.prob), P(self.scale), P(self.k_column), P(self.k_scale), P(self.k_count),
                P(self.kexp) if bal else None, P(self.gshift) if bal else None, st)

    def _plan_small_now(self) -> bool:
        """bmm_plan_small replaces the separate planning kernels: own statistics (no group's
        shared stage or exchange feeding probabilities from elsewhere)."""
        return self.plan_small and self.shared is None and self.exchange is None

    def _contract_sketch(self, M, N, dt, st, planned: bool = False):
        """Compress the drawn sketch (column, scale) and contract it: C @ D.
        planned: bmm_plan_small already compressed it and balanced the exponents."""
        B, m, n, p, W = self.B, self.m, self.n, self.p, self.W
        sM, sN = m * n, n * p
        ldm, ldn = M.stride(-2), N.stride(-2)
        P = lambda t: t.data_ptr()  # noqa: E731
        if self.compress and not planned:
            # duplicates of a column share its scale: contract the distinct columns only
            self._c("bmm_compress_sketch", P(self.column), P(self.scale), W, W, n, B, P(self.ws_cmp),
                    self.ws_cmp.numel(), P(self.k_column), P(self.k_scale), P(self.k_count), st)
        if self.fused:
            # float32 inputs: the split gather runs inside the tcgen05 contraction's producer warps
            self._c("bmm_gemm_f32split_gather", dt, P(M), ldm, sM, P(N), ldn, sN, m, p, P(self.k_column),
                    P(self.k_scale), W, W, P(self.k_count), B, P(self.CD), p, m * p, st)
        elif self.fused16:
            self.fused_f16(M, N, st, balance=not planned)
        elif self.tf32 and self.compress:
            # float32 inputs: split gather + tcgen05 contraction (fp16 or tf32 + bf16 split)
            self.split_gather(M, N, st, balance=not planned)
            self.split_gemm(st)
        elif self.tf32:
            self._c("bmm_gather_f32split", dt, P(M), ldm, sM, P(N), ldn, sN, m, p, P(self.column), P(self.scale), W, W,
                    B, P(self.a_hi), P(self.a_x), P(self.b_hi), P(self.b_x), st)
            self._c("bmm_gemm_f32split", P(self.a_hi), P(self.a_x), P(self.b_hi), P(self.b_x), m, p, W, B,
                    P(self.CD), p, m * p, st)
        else:
            self.contract(M, N, st)
        return self._result()

    def fused_f16(self, M, N, st=None, balance: bool = True):
        """Balanced exponents, then the fp16-split gather + contraction in one
        kernel (K4 + K6 fused, bmm_gemm_f16split_gather)."""
        B, m, n, p, W = self.B, self.m, self.n, self.p, self.W
        st = _lib.stream_ptr() if st is None else st
        P = lambda t: t.data_ptr()  # noqa: E731
        if balance:
            self._c("bmm_balance_f16", P(self.colsq), P(self.rowsq), n, P(self.k_column), P(self.k_scale), W, W,
                    P(self.k_count), B, P(self.kexp), P(self.gshift), st)
        self._c("bmm_gemm_f16split_gather", _lib.matrix_dtype(M), P(M), M.stride(-2), m * n, P(N), N.stride(-2),
                n * p, m, n, p, P(self.k_column), P(self.k_scale), P(self.kexp), P(self.gshift), W, W, P(self.k_count),
                B, P(self.CD), p, m * p, st)

    def split_gather(self, M, N, st=None, balance: bool = True):
        """The float32 path's split gather of the compressed sketch (K4)."""
        B, m, n, p, W = self.B, self.m, self.n, self.p, self.W
        st = _lib.stream_ptr() if st is None else st
        dt = _lib.matrix_dtype(M)
        ldm, ldn = M.stride(-2), N.stride(-2)
        P = lambda t: t.data_ptr()  # noqa: E731
        if self.f16:
            if balance:
                self._c("bmm_balance_f16", P(self.colsq), P(self.rowsq), n, P(self.k_column), P(self.k_scale), W, W,
                        P(self.k_count), B, P(self.kexp), P(self.gshift), st)
            self._c("bmm_gather_f16split_dk", dt, P(M), ldm, m * n, P(N), ldn, n * p, m, p, P(self.k_column),
                    P(self.k_scale), P(self.kexp), P(self.gshift), W, W, P(self.k_count), B, P(self.a_hi),
                    P(self.a_x), P(self.b_hi), P(self.b_x), st)
        else:
            self._c("bmm_gather_f32split_dk", dt, P(M), ldm, m * n, P(N), ldn, n * p, m, p, P(self.k_column),
                    P(self.k_scale), W, W, P(self.k_count), B, P(self.a_hi), P(self.a_x), P(self.b_hi),
                    P(self.b_x), st)

    def split_gemm(self, st=None):
        """The float32 path's tcgen05 contraction of the split operands (K6)."""
        B, m, p, W = self.B, self.m, self.p, self.W
        st = _lib.stream_ptr() if st is None else st
        P = lambda t: t.data_ptr()  # noqa: E731
        if self.f16:
            self._c("bmm_gemm_f16split_dk", P(self.a_hi), P(self.a_x), P(self.b_hi), P(self.b_x), m, p, W,
                    P(self.k_count), P(self.gshift), B, P(self.CD), p, m * p, st)
        else:
            self._c("bmm_gemm_f32split_dk", P(self.a_hi), P(self.a_x), P(self.b_hi), P(self.b_x), m, p, W,
                    P(self.k_count), B, P(self.CD), p, m * p, st)

    def contract(self, M, N, st=None):
        """C @ D of the current sketch on the float64 path (gather + DMMA GEMM, or
        the int8 Ozaki contraction with the gather fused into its digit split)."""
        B, m, n, p, W = self.B, self.m, self.n, self.p, self.W
        st = _lib.stream_ptr() if st is None else st
        dt = _lib.matrix_dtype(M)
        sM, sN = m * n, n * p
        ldm, ldn = M.stride(-2), N.stride(-2)
        P = lambda t: t.data_ptr()  # noqa: E731
        col, sc = (self.k_column, self.k_scale) if self.compress else (self.column, self.scale)
        if self.gemm_engine == "i8":
            kd = P(self.k_count) if self.compress else None
            # balance C's columns against D's rows with the norm pass (exact powers of two)
            self._c("bmm_balance_exponents", P(self.colsq), P(self.rowsq), n, P(col), W, W, kd, B, P(self.kexp), st)
            self._c("bmm_gemm_i8_gather", dt, P(M), ldm, sM, P(N), ldn, sN, P(col), P(sc), P(self.kexp), W, m, p, W,
                    kd, B, P(self.CD), p, m * p, P(self.ws_gemm), self.ws_gemm.numel(), st)
        elif self.compress and self._joint is not None:
            # member of a joint PipelineGroup: gather into the group's pooled operands
            # (row stride ldc); the group contracts every member in one batched GEMM
            ldc = self._joint
            self._c("bmm_gather_dk", dt, _lib.BMM_F64, P(M), ldm, sM, P(N), ldn, sN, m, p, P(self.k_column),
                    P(self.k_scale), W, W, P(self.k_count), B, P(self.C), ldc, m * ldc, P(self.D), p, ldc * p, st)
        elif self.compress:
            self._c("bmm_gather_dk", dt, _lib.BMM_F64, P(M), ldm, sM, P(N), ldn, sN, m, p, P(self.k_column),
                    P(self.k_scale), W, W, P(self.k_count), B, P(self.C), W, m * W, P(self.D), p, W * p, st)
            self._c("bmm_gemm_f64_dk", P(self.C), W, m * W, P(self.D), p, W * p, m, p, W, P(self.k_count), B,
                    P(self.CD), p, m * p, P(self.ws_gemm), self.ws_gemm.numel(), st)
        else:
            self._c("bmm_gather", dt, _lib.BMM_F64, P(M), ldm, sM, P(N), ldn, sN, m, p, P(self.column),
                    P(self.scale), W, W, B, P(self.C), W, m * W, P(self.D), p, W * p, st)
            self._c("bmm_gemm_f64", P(self.C), W, m * W, P(self.D), p, W * p, m, p, W, B, P(self.CD), p, m * p,
                    P(self.ws_gemm), self.ws_gemm.numel(), st)

    def _plan_ssm(self, st):
        """SSM (estimators.py:221-253): q_k from the norm pass, draws from the
        caller's stream, then the whole-block draws expanded to sketch columns."""
        B, n, K = self.B, self.n, self.K
        P = lambda t: t.data_ptr()  # noqa: E731
        self._c("bmm_block_probs", P(self.colsq), P(self.rowsq), n, P(self.offsets), K, B, self.max_len, None, None,
                P(self.fnorm), None, None, st)
        self._c("bmm_normalize", P(self.fnorm), K, B, P(self.q), P(self.status), st)
        self._c("bmm_block_cdf", P(self.q), P(self.qoff), 1, B, K, P(self.qcum), P(self.qlast), st)
        (states,) = self._seedbuf["states"]
        self._c("bmm_sample", P(self.q), P(self.qcum), P(self.qlast), P(self.qoff), 1, B, K, K, P(self.q_bud),
                P(self.q_coloff), self.draws, P(states), P(self.blk), P(self.blk_prob), P(self.blk_scale), st)
        self._c("bmm_expand_blocks", P(self.blk), P(self.blk_scale), self.draws, self.draws, P(self.offsets),
                self.sizes[0], B, P(self.column), P(self.scale), self.W, st)

    def _segsq(self, M, N, dt, k0, k1, B, st):
        """OPL g_k^2 for blocks k0..k1-1 of every problem (k0 > 0: one problem, a
        streamed chunk)."""
        P = lambda t: t.data_ptr()  # noqa: E731
        m, p = self.m, self.p
        sM, sN = m * self.n, self.n * p
        if self.seg_engine == "gram":
            self._c("bmm_segsq_gram", dt, P(M), M.stride(-2), sM, P(N), N.stride(-2), sN, m, p,
                    P(self.offsets) + 8 * k0, k1 - k0, 0, B, P(self.gsq) + 8 * k0, st)
        elif self.seg_engine == "i8":
            n_inner = int(sum(self.sizes[k0:k1]))
            self._c("bmm_segsq_i8", dt, P(M), M.stride(-2), sM, P(N), N.stride(-2), sN, m, p, n_inner,
                    P(self.offsets) + 8 * k0, k1 - k0, 0, B, P(self.gsq) + 8 * k0, P(self.ws_seg),
                    self.ws_seg.numel(), st)
        else:
            A, Bm = self._f64(M, N)
            self._c("bmm_segsq_f64", P(A), A.stride(-2), sM, P(Bm), Bm.stride(-2), sN, m, p,
                    P(self.offsets) + 8 * k0, k1 - k0, 0, B, P(self.gsq) + 8 * k0, P(self.ws_seg),
                    self.ws_seg.numel(), st)
        if getattr(self, "exchange", None) is not None and k0 == 0 and k1 == self.K:
            self.exchange.sum_(self.gsq)  # C2: ||M^k N_k||_F^2 is the sum over the output tiles

    def _f64(self, M, N):
        if M.dtype == torch.float64:
            return M, N
        if getattr(self, "_up", None) is None or self._up[0].shape != M.shape:
            self._up = (torch.empty(M.shape, dtype=torch.float64, device=M.device),
                        torch.empty(N.shape, dtype=torch.float64, device=N.device))
        self._up[0].copy_(M)
        self._up[1].copy_(N)
        return self._up

    def check(self) -> None:
        """Raise the reference's exception for the first failing problem (syncs)."""
        st = self.status.cpu().numpy()
        bad = np.flatnonzero(st != 0)
        if bad.size:
            b = int(bad[0])
            if self.method == "SSM" and int(st[b]) == _lib.ST_ZERO_SCORE:
                raise ValueError("all blocks have zero norm: nothing to sample")  # plan.py:494-495
            raise_status(int(st[b]), int(self.diag[b].item()), self.c)

    # audit views
    def budgets_host(self) -> np.ndarray:
        return self.budgets.view(self.B, self.K).cpu().numpy()

    def columns_host(self) -> np.ndarray:
        if self.method == "SSM":
            return self.blk.view(self.B, self.draws).cpu().numpy()
        return self.column.view(self.B, self.W).cpu().numpy()

    def scales_host(self) -> np.ndarray:
        if self.method == "SSM":
            return self.blk_scale.view(self.B, self.draws).cpu().numpy()
        return self.scale.view(self.B, self.W).cpu().numpy()


class SharedStats:
    """The statistics every member of a PipelineGroup over one instance (same M,
    N, partition, batch and dtype) would otherwise recompute: the norm pass,
    the optimal probabilities, score sums and main CDF, and (when a member is
    OPL) the block-product norms g_k^2.  The reference recomputes them inside
    every allocator call (plan.py:165-189, reached from allocate_* 383-480);
    here one stage computes them once per group call and the members read the
    same buffers (they only read them: UU keeps its own CDF, SSM its own block
    probabilities)."""

    _c = None  # bound below to SketchPipeline's launch helpers
    _segsq = None
    _f64 = None

    def __init__(self, pipes):
        p0 = pipes[0]
        key = lambda q: (q.m, q.n, q.p, q.sizes, q.B, q.dtype, q.colsq.device)  # noqa: E731
        if any(key(q) != key(p0) for q in pipes):
            raise ValueError("shared statistics need members over one instance (shape, partition, batch, dtype)")
        self.lib = p0.lib
        self.m, self.n, self.p, self.B, self.K = p0.m, p0.n, p0.p, p0.B, p0.K
        self.sizes, self.max_len, self.offsets = p0.sizes, p0.max_len, p0.offsets
        self.timeline, self.stamps = None, None
        self.exchange = p0.exchange
        if any(q.exchange is not p0.exchange for q in pipes):
            raise ValueError("shared statistics need one exchange for every member")
        self.colsq, self.rowsq = p0.colsq, p0.rowsq
        self.needs_probs = any(q.method not in ("SSM", "UU") for q in pipes)
        opl = [q for q in pipes if q.method == "OPL"]
        self.needs_gsq = bool(opl)
        src = next((q for q in pipes if q.method not in ("SSM", "UU")), p0)
        self.probs, self.s, self.cum, self.last = src.probs, src.s, src.cum, src.last
        self.seg_engine = None
        if opl:
            self.gsq, self.seg_engine, self.ws_seg = opl[0].gsq, opl[0].seg_engine, opl[0].ws_seg
        for q in pipes:
            q.colsq, q.rowsq = self.colsq, self.rowsq
            if q.method not in ("SSM", "UU"):
                q.probs, q.s, q.cum, q.last = self.probs, self.s, self.cum, self.last
            if q.method == "OPL":
                q.gsq = self.gsq
            q.shared = self

    def launch_probs(self, M: torch.Tensor, N: torch.Tensor, chunks=None) -> bool:
        """Norm pass (+ g_k^2 per chunk when chunked, or with the norms fused into
        the Gram kernel) and the block probabilities.  True when g_k^2 is done."""
        return _stats_launch(self, M, N, chunks, probs=self.needs_probs, gsq=self.needs_gsq)

    def fused(self, M: torch.Tensor) -> bool:
        """g_k^2 and the norm pass in one kernel (launch_probs does both)."""
        return self.needs_gsq and _fused_stats(self, M)

    def launch_gsq(self, M: torch.Tensor, N: torch.Tensor) -> None:
        if self.needs_gsq:
            self._segsq(M, N, _lib.matrix_dtype(M), 0, self.K, self.B, _lib.stream_ptr())


SharedStats._c = SketchPipeline._c
SharedStats._segsq = SketchPipeline._segsq
SharedStats._f64 = SketchPipeline._f64


class PipelineGroup:
    """Independent pipelines over the same inputs (e.g. a c x method sweep, the
    reference's bench loop ``bench.py:209-245``) replayed as ONE CUDA graph whose
    branches run concurrently: each pipeline is captured on its own forked
    stream, so one product's latency-bound planning kernels overlap another's
    GEMM. Results are those of the member pipelines run one after another.

    shared (default on, BMM_SHARED=0 disables): members over one instance read
    one SharedStats stage -- the norm pass, block probabilities and g_k^2 run
    once per call instead of once per member (bit-identical: the same kernels on
    the same inputs).  joint: see below."""

    def __init__(self, pipes, joint=None, shared=None):
        self.pipes = list(pipes)
        self.graph = None
        self.graph_launches = 0
        if shared is None:
            shared = os.environ.get("BMM_SHARED", "1") != "0"
        p0 = self.pipes[0] if self.pipes else None
        key = lambda q: (q.m, q.n, q.p, q.sizes, q.B, q.dtype, q.colsq.device)  # noqa: E731
        self.shared = None
        if shared and len(self.pipes) > 1 and all(key(q) == key(p0) for q in self.pipes):
            self.shared = SharedStats(self.pipes)
        # joint contraction: float64 compressed members on the DMMA engine with one output
        # shape gather into pooled operands, and ONE batched GEMM contracts all of them
        # (per-member inner lengths read on the device).  Nine 500 x ~3000 x 500 products
        # then fill the GPU with their own tiles instead of split-K partials.
        # BMM_JOINT=0 (or joint=False) keeps one GEMM per member.
        if joint is None:
            joint = os.environ.get("BMM_JOINT", "1") != "0"
        self.joint = bool(joint) and len(self.pipes) > 1 and all(
            q.B == 1 and not q.tf32 and q.compress and q.gemm_engine == "dmma"
            and (q.m, q.p) == (p0.m, p0.p) and q.C.device == p0.C.device for q in self.pipes)
        self._jgroups = []
        if self.joint:
            # one batched GEMM per sketch width: its members finish planning at about the
            # same time, and each width's GEMM can start while the other widths still plan
            m, p, dev = p0.m, p0.p, p0.C.device
            f64 = dict(dtype=torch.float64, device=dev)
            # BMM_JOINT_BY=method pools each method's members instead (pool width = the
            # widest member; per-member inner lengths are read on the device anyway)
            by = os.environ.get("BMM_JOINT_BY", "width")
            by_w = {}
            for i, q in enumerate(self.pipes):
                by_w.setdefault(q.method if by == "method" else q.W, []).append(i)
            for key, idx in by_w.items():
                Wj = max(self.pipes[i].W for i in idx)
                G = len(idx)
                jg = dict(idx=idx, W=Wj, C=torch.zeros((G, m, Wj), **f64), D=torch.zeros((G, Wj, p), **f64),
                          k=torch.zeros(G, dtype=torch.int64, device=dev), CD=torch.empty((G, m, p), **f64),
                          ws=torch.empty(max(256, p0.lib.bmm_gemm_f64_workspace(m, p, Wj, G)), dtype=torch.uint8,
                                         device=dev))
                for j, i in enumerate(idx):
                    q = self.pipes[i]
                    q.C, q.D = jg["C"][j].view(-1), jg["D"][j].view(-1)
                    q.k_count, q.CD = jg["k"][j:j + 1], jg["CD"][j].view(-1)
                    q._joint = Wj
                    del q.ws_gemm
                self._jgroups.append(jg)

    def _active(self, on: bool) -> None:
        for q in self.pipes:
            q._group_active = on

    def _joint_gemm(self, jg=None) -> None:
        m, p = self.pipes[0].m, self.pipes[0].p
        for g in ([jg] if jg is not None else self._jgroups):
            G, Wj = len(g["idx"]), g["W"]
            _lib.call("bmm_gemm_f64_dk", g["C"].data_ptr(), Wj, m * Wj, g["D"].data_ptr(), p, Wj * p, m, p, Wj,
                      g["k"].data_ptr(), G, g["CD"].data_ptr(), p, m * p, g["ws"].data_ptr(), g["ws"].numel(),
                      _lib.stream_ptr())

    def serial(self) -> bool:
        """BMM_GROUP_SERIAL=1: members one after another (one stream, OPL last)
        instead of concurrent branches.  Measured at config 4, where every
        member's contraction alone fills the GPU: 177.5 vs 180.0 ms per step and a
        longer single-step latency end to end (808 vs 770 ms), i.e. within the
        run-to-run spread, so concurrent branches stay the default."""
        forced = os.environ.get("BMM_GROUP_SERIAL", "")
        return forced == "1"

    def _branch_streams(self) -> list:
        """One stream per member.  OPL members (the longest chains: their g_k
        contraction occupies every SM) get the high priority, so their kernels take
        SMs first and the other branches fill the gaps (BMM_BRANCH_PRIORITY=0: all
        equal).  Serial groups: ONE stream, members needing g_k last."""
        if self.serial():
            one = torch.cuda.Stream()
            return [one for _ in self.pipes]
        mode = os.environ.get("BMM_BRANCH_PRIORITY", "2")
        if mode == "0":
            return [torch.cuda.Stream() for _ in self.pipes]
        # "2" (default): the two-step members too -- with the statistics shared, their
        # pilot chains (pilot plan, draws, pilot norms, main plan) are the longest
        hi = ("OPL",) if mode == "1" else ("OPL", "ONU", "ONMCNR")
        return [torch.cuda.Stream(priority=-1 if q.method in hi else 0) for q in self.pipes]

    def _order(self) -> list:
        """Member launch order: as given, except serial groups put OPL (which waits
        for the shared g_k) after the others."""
        idx = list(range(len(self.pipes)))
        if self.serial():
            idx.sort(key=lambda i: self.pipes[i].method == "OPL")
        return idx

    def _launch_all(self, M: torch.Tensor, N: torch.Tensor) -> None:
        self._active(True)
        try:
            if self.shared is not None:
                if not self.shared.launch_probs(M, N):
                    self.shared.launch_gsq(M, N)
            for pipe in self.pipes:
                pipe.launch(M, N)
            if self.joint:
                self._joint_gemm()
        finally:
            self._active(False)

    def _fork_gsq(self) -> bool:
        """g_k^2 beside the norm pass on its own stream?  Small instances (config 2:
        the two fill the GPU together) gain; at config 4 both are full-GPU kernels
        and the interleaved CTAs cost more than they overlap (tools/timeline.py
        cfg4: statistics done at 40.7 ms forked vs 38.8 ms in sequence).
        BMM_GSQ_FORK=0|1 forces either."""
        forced = os.environ.get("BMM_GSQ_FORK", "")
        if forced in ("0", "1"):
            return forced == "1"
        sh = self.shared
        return sh.B * sh.m * sh.n < (1 << 30)

    def _fork_stats(self, cap, M, N, chunks=None):
        """Enqueue the shared statistics on their own streams (forked from `cap`):
        the norm pass and block probabilities on one, OPL's g_k^2 (which needs only
        M and N) concurrently on another.  Returns (event after the probabilities,
        event after probabilities AND g_k^2, the joined stream)."""
        ss = torch.cuda.Stream(priority=-1)
        ss.wait_stream(cap)
        ev_p, ev_g = torch.cuda.Event(), torch.cuda.Event()
        gs = None
        fused = chunks is None and self.shared.fused(M)
        if chunks is None and self.shared.needs_gsq and not fused and self._fork_gsq():
            gs = torch.cuda.Stream(priority=-1)
            gs.wait_stream(cap)
            with torch.cuda.stream(gs):
                self.shared.launch_gsq(M, N)
        with torch.cuda.stream(ss):
            self.shared.launch_probs(M, N, chunks)  # chunked: g_k^2 per landed chunk in here
            ev_p.record(ss)
            if gs is not None:
                ss.wait_stream(gs)
            elif chunks is None and self.shared.needs_gsq and not fused:  # not forked: after the probabilities
                self.shared.launch_gsq(M, N)
            ev_g.record(ss)
        return ev_p, ev_g, ss

    def _member_wait(self, s, pipe, evs):
        if evs is not None:
            s.wait_event(evs[1] if pipe.method == "OPL" else evs[0])

    def capture(self, M: torch.Tensor, N: torch.Tensor) -> None:
        if any(q.exchange is not None for q in self.pipes):
            raise RuntimeError("sharded members exchange through host collectives: run them eagerly")
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):  # warm-up: lazy buffers outside the capture
            self._launch_all(M, N)
        cur.wait_stream(side)
        streams = self._branch_streams()
        g = torch.cuda.CUDAGraph()
        n0 = _lib.launches()
        self._active(True)
        try:
            with torch.cuda.graph(g):
                cap = torch.cuda.current_stream()
                evs = None
                extra = []
                if self.shared is not None:
                    *evs, ss = self._fork_stats(cap, M, N)
                    extra.append(ss)
                for i in self._order():
                    s, pipe = streams[i], self.pipes[i]
                    s.wait_stream(cap)
                    self._member_wait(s, pipe, evs)
                    with torch.cuda.stream(s):
                        pipe.launch(M, N)
                for jg in self._jgroups:  # each width's GEMM after its own members
                    js = torch.cuda.Stream()
                    for i in jg["idx"]:
                        js.wait_stream(streams[i])
                    with torch.cuda.stream(js):
                        self._joint_gemm(jg)
                    extra.append(js)
                for s in list(dict.fromkeys(streams)) + extra:  # serial groups share one stream
                    cap.wait_stream(s)
        finally:
            self._active(False)
        self.graph_launches = _lib.launches() - n0
        self.graph, self._graph_ptrs = g, (M.data_ptr(), N.data_ptr())

    def capture_host(self, M: torch.Tensor, N: torch.Tensor, M_host: torch.Tensor, N_host: torch.Tensor,
                     out_host: list, seeds: list, n_chunks: int = 8) -> None:
        """End-to-end graph from pinned host inputs to pinned host products: M's
        block-column slabs and N's row slabs are copied chunk by chunk on a copy
        stream, the norm pass (and OPL segmented square sums) runs on each chunk as
        it lands, then the rest of every member's pipeline, then each product is
        copied back.  Replay with run_host().  Single problem (batch 1), float64
        or float32 inputs."""
        pipes = self.pipes
        sizes = pipes[0].sizes
        n, m, p = pipes[0].n, pipes[0].m, pipes[0].p
        es = M.element_size()
        off = np.concatenate([[0], np.cumsum(sizes)])
        bounds = [0]
        for c in range(1, n_chunks):
            k = int(np.searchsorted(off, c * n / n_chunks))
            if bounds[-1] < k < len(sizes):
                bounds.append(k)
        bounds.append(len(sizes))
        plan = [(int(off[k0]), int(off[k1]), k0, k1) for k0, k1 in zip(bounds[:-1], bounds[1:])]
        for pipe, sd in zip(pipes, seeds):  # seed buffers exist before the warm-up and the capture
            pipe.set_seeds(sd)
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):  # warm-up: lazy buffers outside the capture
            self._launch_all(M, N)
        cur.wait_stream(side)
        copy = torch.cuda.Stream()
        streams = self._branch_streams()
        g = torch.cuda.CUDAGraph()
        n0 = _lib.launches()
        self._active(True)
        try:
            with torch.cuda.graph(g):
                cap = torch.cuda.current_stream()
                copy.wait_stream(cap)
                chunks = []
                with torch.cuda.stream(copy):
                    cs = _lib.stream_ptr()
                    for c0, c1, k0, k1 in plan:
                        _lib.call("bmm_copy2d", M.data_ptr() + es * c0, es * n, M_host.data_ptr() + es * c0, es * n,
                                  es * (c1 - c0), m, 1, cs)
                        nb = es * (c1 - c0) * p
                        _lib.call("bmm_copy2d", N.data_ptr() + es * c0 * p, nb, N_host.data_ptr() + es * c0 * p, nb,
                                  nb, 1, 1, cs)
                        ev = torch.cuda.Event()
                        ev.record(copy)
                        chunks.append((c0, c1, k0, k1, ev))
                evs, extra = None, [copy]
                if self.shared is not None:
                    *evs, ss = self._fork_stats(cap, M, N, chunks)
                    extra.append(ss)
                for i in self._order():
                    s, pipe, oh = streams[i], pipes[i], out_host[i]
                    s.wait_stream(cap)
                    self._member_wait(s, pipe, evs)
                    with torch.cuda.stream(s):
                        if self.shared is not None:
                            out = pipe.launch(M, N)
                        else:
                            out = pipe.launch(M, N, chunks=chunks)
                        if not self.joint:
                            oh.copy_(out.reshape(oh.shape), non_blocking=True)
                for jg in self._jgroups:  # joint mode: each width's GEMM, then its products go home
                    js = torch.cuda.Stream()
                    for i in jg["idx"]:
                        js.wait_stream(streams[i])
                    with torch.cuda.stream(js):
                        self._joint_gemm(jg)
                        for j, i in enumerate(jg["idx"]):
                            out_host[i].copy_(jg["CD"][j].reshape(out_host[i].shape), non_blocking=True)
                    extra.append(js)
                for s in list(dict.fromkeys(streams)) + extra:
                    cap.wait_stream(s)
        finally:
            self._active(False)
        self.host_graph_launches = _lib.launches() - n0
        self.host_graph = g

    def run_host(self, seeds: list) -> None:
        """Replay the end-to-end graph (capture_host); products land in out_host."""
        for pipe, s in zip(self.pipes, seeds):
            pipe.set_seeds(s)
        self.host_graph.replay()

    def run(self, M: torch.Tensor, N: torch.Tensor, seeds: list) -> list:
        """One call per member pipeline (same seeds contract as SketchPipeline.run)."""
        for pipe, s in zip(self.pipes, seeds):
            pipe.set_seeds(s)
        if self.graph is None or self._graph_ptrs != (M.data_ptr(), N.data_ptr()):
            self._launch_all(M, N)
        else:
            self.graph.replay()
        return [pipe._result() for pipe in self.pipes]

    def check(self) -> None:
        for pipe in self.pipes:
            pipe.check()
