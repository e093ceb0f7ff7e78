"""Monte Carlo replication engine -- SURVEY.md §8(f1).

The reference validates its bounds by repeating ``estimate_product`` on one
instance hundreds to thousands of times (``coverage_check``
analysis.py:343-366, ``coverage_check_plan`` :369-380,
``normality_diagnostic`` :390-416; the bench rep loop bench.py:258-278).
Every replication re-runs the whole Python path.  Here one plan is uploaded
once (probabilities, CDF tables, budgets) and the replications run as a
batch on the device:

    rng.spawn(R) -> per-replication SeedSequence words          (host, O(R))
    bmm_seed_streams   R x K child PCG64 streams                 (device)
    bmm_sample_reps    draws of all replications, shared plan    (device)
    bmm_gather         C_r, D_r with zero input strides          (device)
    bmm_gemm_f64       batched C_r @ D_r (DMMA)                  (device)
    bmm_sqdiff         ||C_r D_r - MN||_F^2 per replication      (device)

Replication r draws exactly what ``estimate_product(M, N, plan, stream_r)``
draws for ``stream_r = rng.spawn(R)[r]`` (bit-identical columns and scales),
and ``rng`` is left with the spawn counter the reference leaves.
"""
from __future__ import annotations

import math
from typing import Callable, NamedTuple, Optional

import numpy as np
import torch

from . import _lib
from . import rng as _rng
from .analysis import sq_diff
from .matrix import multiply_exact
from .plan import DeviceInstance, SamplingPlan


class CoverageResult(NamedTuple):
    """analysis.py:327-332."""

    reps: int
    violations: int
    frequency: float
    ci_low: float
    ci_high: float


class NormalityResult(NamedTuple):
    """analysis.py:383-387."""

    samples: np.ndarray
    mean: float
    variance: float
    ks_distance: float


def clopper_pearson(k: int, n: int, confidence: float = 0.95) -> tuple[float, float]:
    """Exact binomial interval (analysis.py:335-340): beta quantiles."""
    from scipy.stats import beta

    alpha = 1.0 - confidence
    lo = 0.0 if k == 0 else float(beta.ppf(alpha / 2, k, n - k + 1))
    hi = 1.0 if k == n else float(beta.ppf(1 - alpha / 2, k + 1, n - k))
    return lo, hi


class ReplicationEngine:
    """Batched replications of ``estimate_product(M, N, plan, stream)``.

    ``chunk`` bounds the replications resident at once (sketch factors are
    m x W and W x p float64 per replication); by default it is sized to
    ``mem_bytes`` of HBM."""

    def __init__(self, M, N, plan: SamplingPlan, chunk: Optional[int] = None, mem_bytes: int = 8 << 30):
        self.plan = plan
        part = plan.partition
        self.inst = inst = DeviceInstance(M, N, part)
        self.K, self.n = inst.K, inst.n
        self.m, self.p = int(inst.M.shape[0]), int(inst.N.shape[1])
        dev = inst.M.device
        self.probs = _lib.f64(plan.probs.flat())
        self.cum = torch.empty(self.n, dtype=torch.float64, device=dev)
        self.last = torch.empty(self.K, dtype=torch.int64, device=dev)
        _lib.call("bmm_block_cdf", _lib.ptr(self.probs), _lib.ptr(inst.offsets), self.K, 1, self.n,
                  _lib.ptr(self.cum), _lib.ptr(self.last), _lib.stream_ptr())
        budgets = np.asarray(plan.budgets, dtype=np.int64)
        col_off = np.zeros(self.K + 1, dtype=np.int64)
        np.cumsum(budgets, out=col_off[1:])
        self.W = int(col_off[-1])
        self.budgets = _lib.i64(budgets)
        self.col_off = _lib.i64(col_off)
        per_rep = 8 * (self.m * self.W + self.W * self.p + self.m * self.p) + 8 * 3 * self.W + 32 * self.K
        self.chunk = int(chunk) if chunk else max(1, int(mem_bytes // max(per_rep, 1)))
        self._exact = None

    @property
    def exact(self) -> torch.Tensor:
        if self._exact is None:
            self._exact = multiply_exact(self.inst.M, self.inst.N)
        return self._exact

    def _stream_words(self, rng, reps: int):
        base, first = _rng.spawn_words(rng, reps)  # rng.spawn(reps): advances the parent counter
        if first + reps > 0xFFFFFFFF:
            raise ValueError("spawn counter beyond one 32-bit key word is not supported")
        return base, first

    def run(self, rng: np.random.Generator, reps: int, *, sq_errors: bool = True,
            entry: Optional[tuple[int, int]] = None, keep_columns: bool = False) -> dict:
        """Run ``reps`` replications on ``rng.spawn(reps)``; returns device
        tensors: ``sq_error`` (reps,) = ||C_r D_r - MN||_F^2, ``entry`` (reps,)
        = (C_r D_r)[h, f], ``columns`` (reps, W) when asked."""
        reps = int(reps)
        if reps < 1:
            raise ValueError("reps must be >= 1")
        base, first = self._stream_words(rng, reps)
        m, p, W, K, n = self.m, self.p, self.W, self.K, self.n
        inst = self.inst
        dev = inst.M.device
        out = {}
        if sq_errors:
            out["sq_error"] = torch.empty(reps, dtype=torch.float64, device=dev)
        if entry is not None:
            h, f = int(entry[0]), int(entry[1])
            if not (0 <= h < m and 0 <= f < p):
                raise IndexError(f"entry {entry} outside the {m}x{p} product")
            out["entry"] = torch.empty(reps, dtype=torch.float64, device=dev)
        if keep_columns:
            out["columns"] = torch.empty((reps, W), dtype=torch.int64, device=dev)
        if W == 0:
            raise ValueError("plan has no draws")
        R = min(self.chunk, reps)
        nw = base.size + 1
        words = np.empty((R, nw), dtype=np.uint32)
        words[:, :-1] = base
        states = torch.empty(R * K * 4, dtype=torch.int64, device=dev)
        column = torch.empty(R * W, dtype=torch.int64, device=dev)
        prob = torch.empty(R * W, dtype=torch.float64, device=dev)
        scale = torch.empty(R * W, dtype=torch.float64, device=dev)
        C = torch.empty(R * m * W, dtype=torch.float64, device=dev)
        D = torch.empty(R * W * p, dtype=torch.float64, device=dev)
        CD = torch.empty(R * m * p, dtype=torch.float64, device=dev)
        first_d = torch.zeros(R, dtype=torch.int64, device=dev)
        lib = _lib.load()
        ws_g = _lib.workspace(max(lib.bmm_gemm_f64_workspace(m, p, W, R), lib.bmm_gemm_f64_err_workspace(m, p, W, R)))
        err = torch.empty(R, dtype=torch.float64, device=dev)
        need_cd = entry is not None  # the products themselves are only read for the entry diagnostic
        exact = self.exact if sq_errors else None
        dt = _lib.matrix_dtype(inst.M)
        st = _lib.stream_ptr()
        for r0 in range(0, reps, R):
            Rc = min(R, reps - r0)
            words[:Rc, -1] = np.arange(first + r0, first + r0 + Rc, dtype=np.int64).astype(np.uint32)
            words_d = torch.as_tensor(words[:Rc].view(np.int32), device=dev)
            _lib.call("bmm_seed_streams", _lib.ptr(words_d), nw, _lib.ptr(first_d), K, Rc, _lib.ptr(states), st)
            _lib.call("bmm_sample_reps", _lib.ptr(self.probs), _lib.ptr(self.cum), _lib.ptr(self.last),
                      _lib.ptr(inst.offsets), K, Rc, n, inst.max_len, _lib.ptr(self.budgets),
                      _lib.ptr(self.col_off), W, _lib.ptr(states), _lib.ptr(column), _lib.ptr(prob),
                      _lib.ptr(scale), st)
            _lib.call("bmm_gather", dt, _lib.BMM_F64, _lib.ptr(inst.M), inst.M.stride(0), 0, _lib.ptr(inst.N),
                      inst.N.stride(0), 0, m, p, _lib.ptr(column), _lib.ptr(scale), W, W, Rc, _lib.ptr(C), W, m * W,
                      _lib.ptr(D), p, W * p, st)
            if sq_errors:
                # K9: ||C_r D_r - MN||_F^2 in the contraction's epilogue; C_r D_r stays on chip
                _lib.call("bmm_gemm_f64_err", _lib.ptr(C), W, m * W, _lib.ptr(D), p, W * p, m, p, W, Rc,
                          _lib.ptr(exact), exact.stride(0), 0, _lib.ptr(CD) if need_cd else None, p, m * p,
                          _lib.ptr(err), _lib.ptr(ws_g), ws_g.numel(), st)
                out["sq_error"][r0:r0 + Rc] = err[:Rc]
            else:
                _lib.call("bmm_gemm_f64", _lib.ptr(C), W, m * W, _lib.ptr(D), p, W * p, m, p, W, Rc, _lib.ptr(CD), p,
                          m * p, _lib.ptr(ws_g), ws_g.numel(), st)
            if entry is not None:
                out["entry"][r0:r0 + Rc] = CD.view(R, m, p)[:Rc, h, f]
            if keep_columns:
                out["columns"][r0:r0 + Rc] = column.view(R, W)[:Rc]
        # the last chunk's device buffers (for kernel timing / inspection)
        self.last_chunk = {"C": C, "D": D, "CD": CD, "ws_gemm": ws_g, "reps": Rc, "column": column, "scale": scale}
        return out


# ---------------------------------------------------------------- reference API

def coverage_check(M, N, reps: int, rng: np.random.Generator,
                   runner: Callable[[np.random.Generator], tuple]) -> CoverageResult:
    """analysis.py:343-366 with a caller-supplied runner(stream) ->
    (estimate, squared-error bound); exact product and errors on device."""
    if reps < 100:
        raise ValueError("need at least 100 replications for a meaningful frequency")
    exact = multiply_exact(_lib.float_matrix(M), _lib.float_matrix(N))
    violations = 0
    for stream in rng.spawn(reps):
        estimate, sq_bound = runner(stream)
        err, _ = sq_diff(estimate, exact)
        if err > sq_bound:
            violations += 1
    lo, hi = clopper_pearson(violations, reps)
    return CoverageResult(reps, violations, violations / reps, lo, hi)


def coverage_check_plan(M, N, plan: SamplingPlan, sq_error_bound: float, reps: int,
                        rng: np.random.Generator) -> CoverageResult:
    """analysis.py:369-380: ``reps`` replications of estimate_product under a
    fixed plan against one bound -- batched on device (ReplicationEngine)."""
    if reps < 100:
        raise ValueError("need at least 100 replications for a meaningful frequency")
    eng = ReplicationEngine(M, N, plan)
    err = eng.run(rng, reps)["sq_error"]
    violations = int((err > float(sq_error_bound)).sum().item())
    lo, hi = clopper_pearson(violations, reps)
    return CoverageResult(reps, violations, violations / reps, lo, hi)


def normality_diagnostic(M, N, plan: SamplingPlan, entry: tuple[int, int], reps: int,
                         rng: np.random.Generator) -> NormalityResult:
    """analysis.py:390-416: standardized errors of one entry over ``reps``
    replications (device batch) and their KS distance from N(0, 1)."""
    from scipy.special import ndtr

    from .variance import elementwise_variance

    if reps < 1000:
        raise ValueError("need at least 1000 replications for the diagnostic")
    h, f = entry
    sigma_sq = float(_lib.host(elementwise_variance(_lib.float_matrix(M), _lib.float_matrix(N), plan))[h, f])
    if sigma_sq <= 0.0:
        raise ValueError(f"entry {entry} has zero variance under this plan")
    eng = ReplicationEngine(M, N, plan)
    exact = float(eng.exact[h, f].item())
    scale = math.sqrt(sigma_sq)
    vals = _lib.host(eng.run(rng, reps, sq_errors=False, entry=(h, f))["entry"])
    samples = (vals - exact) / scale
    z = np.sort(samples)
    cdf = ndtr(z)
    grid = np.arange(1, reps + 1) / reps
    ks = float(max((grid - cdf).max(), (cdf - (grid - 1.0 / reps)).max()))
    return NormalityResult(samples, float(samples.mean()), float(samples.var(ddof=1)), ks)
