"""High-probability error bounds and the analytics CSV (analysis.py:127-316,
419-470) -- the closed-form layer the Monte Carlo coverage checks validate.

Everything here is scalar/K-length arithmetic on quantities the device
computes (score sums s_k, block-product norms g_k, probabilities, Frobenius
norms); it mirrors the reference's formulas and error behaviour.
"""
from __future__ import annotations

import csv
import math
from dataclasses import dataclass
from typing import NamedTuple, Optional, Sequence

import numpy as np

from .matrix import BlockPartition, frobenius_norm
from .plan import SamplingPlan, block_scores, optimal_probabilities, prob_floor_ratio, score_sums

DEGENERATE_TOL = 1e-12


@dataclass(frozen=True, eq=False)
class CancellationStats:
    """Per-block g_k/s_k ratios and cancellation statistics (analysis.py:127-145)."""

    ratios: np.ndarray
    cancel: np.ndarray
    cancel_lo: float
    cancel_hi: float
    lo_available: bool
    exact: bool
    zero_score_blocks: tuple
    degenerate_blocks: tuple


def cancellation_stats(M, N, part: BlockPartition, pilot_norms=None,
                       degenerate_tol: float = DEGENERATE_TOL) -> CancellationStats:
    """analysis.py:148-196; exact g_k from the DMMA segmented square sums,
    or the given pilot norms (cancellation then under an absolute value)."""
    s = np.asarray(score_sums(M, N, part), dtype=np.float64)
    if (s == 0).all():
        raise ValueError("all blocks have zero score")
    if pilot_norms is not None:
        g = np.asarray(pilot_norms, dtype=np.float64)
        if g.shape != s.shape:
            raise ValueError("need one pilot norm per block")
        exact = False
    else:
        g = block_scores(M, N, part).product_norms
        exact = True
    ratios = np.full(part.num_blocks, np.nan)
    inc = s > 0
    ratios[inc] = g[inc] / s[inc]
    cancel = 1.0 - ratios ** 2
    if not exact:
        cancel = np.abs(cancel)
    degenerate = inc & ((ratios >= 1.0 - degenerate_tol) if exact else (cancel <= degenerate_tol))
    usable = inc & ~degenerate
    hi = float(np.nanmax(cancel[inc])) if inc.any() else 0.0
    lo, lo_ok = (float(cancel[usable].min()), True) if usable.any() else (0.0, False)
    return CancellationStats(ratios, cancel, lo, max(hi, 0.0), lo_ok, exact,
                             tuple(np.where(~inc)[0]), tuple(np.where(degenerate)[0]))


@dataclass(frozen=True, eq=False)
class BoundInputs:
    """analysis.py:199-229."""

    c: int
    fail_prob: float
    prob_floor: float
    cancel_lo: float
    cancel_hi: float
    frob_m: float
    frob_n: float
    ratios: Optional[np.ndarray] = None
    cancel_hi_exact: Optional[float] = None

    def __post_init__(self):
        if self.c < 1:
            raise ValueError("c must be >= 1")
        if not 0.0 < self.fail_prob < 1.0:
            raise ValueError("fail_prob must lie in (0, 1)")
        if not 0.0 <= self.prob_floor <= 1.0 + 1e-12:
            raise ValueError("prob_floor must lie in [0, 1]")
        if self.cancel_lo < 0 or self.cancel_hi < self.cancel_lo - 1e-15:
            raise ValueError("need 0 <= cancel_lo <= cancel_hi")
        if self.frob_m < 0 or self.frob_n < 0:
            raise ValueError("norms must be >= 0")


class BoundPair(NamedTuple):
    variance_bound: float
    sq_error_bound: float


def _base(inp: BoundInputs) -> float:
    return inp.frob_m ** 2 * inp.frob_n ** 2 / (inp.prob_floor * inp.c)


def _tail(inp: BoundInputs) -> float:
    return math.sqrt((8.0 / inp.prob_floor) * math.log(1.0 / inp.fail_prob))


def bounds_optimal_allocation(inp: BoundInputs) -> BoundPair:
    """analysis.py:241-254."""
    lo, hi, fl = inp.cancel_lo, inp.cancel_hi, inp.prob_floor
    if fl <= 0.0 or lo <= 0.0:
        return BoundPair(math.inf, math.inf)
    phi = math.sqrt(hi - lo * fl + hi * lo * fl) / (hi * lo) ** 0.25
    eta = phi + math.sqrt(hi / lo) * _tail(inp)
    return BoundPair(phi ** 2 * _base(inp), eta ** 2 * _base(inp))


def bounds_score_allocation(inp: BoundInputs) -> BoundPair:
    """analysis.py:257-268."""
    hi, fl = inp.cancel_hi, inp.prob_floor
    if not 0.0 <= hi <= 1.0 + 1e-12:
        raise ValueError("score-allocation bound needs an exact high statistic in [0, 1]")
    if fl <= 0.0:
        return BoundPair(math.inf, math.inf)
    phi = math.sqrt(max(1.0 - fl * (1.0 - hi), 0.0))
    eta = phi + _tail(inp)
    return BoundPair(phi ** 2 * _base(inp), eta ** 2 * _base(inp))


def bounds_pilot_allocation(inp: BoundInputs) -> BoundPair:
    """analysis.py:271-283."""
    if inp.cancel_hi_exact is None:
        raise ValueError("pilot bound needs cancel_hi_exact")
    lo, hi, hx, fl = inp.cancel_lo, inp.cancel_hi, inp.cancel_hi_exact, inp.prob_floor
    if fl <= 0.0 or lo <= 0.0:
        return BoundPair(math.inf, math.inf)
    phi = math.sqrt(hi - lo * fl + hx * lo * fl) / (hi * lo) ** 0.25
    eta = phi + math.sqrt(hi / lo) * _tail(inp)
    return BoundPair(phi ** 2 * _base(inp), eta ** 2 * _base(inp))


def bound_inputs_for_plan(M, N, plan: SamplingPlan, fail_prob: float,
                          degenerate_tol: float = DEGENERATE_TOL) -> BoundInputs:
    """analysis.py:286-315."""
    part = plan.partition
    ex = cancellation_stats(M, N, part, degenerate_tol=degenerate_tol)
    floor = prob_floor_ratio(plan.probs, optimal_probabilities(M, N, part))
    if plan.pilot_norms is not None:
        st = cancellation_stats(M, N, part, pilot_norms=plan.pilot_norms, degenerate_tol=degenerate_tol)
        hx = ex.cancel_hi
    else:
        st, hx = ex, None
    return BoundInputs(c=plan.total, fail_prob=fail_prob, prob_floor=0.0 if floor.support_mismatch else floor.ratio,
                       cancel_lo=st.cancel_lo if st.lo_available else 0.0, cancel_hi=st.cancel_hi,
                       frob_m=frobenius_norm(M), frob_n=frobenius_norm(N), ratios=st.ratios,
                       cancel_hi_exact=hx)


@dataclass(frozen=True)
class AnalyticsRow:
    """analysis.py:419-432."""

    instance: str
    method: str
    c: int
    num_blocks: int
    objective: float
    sq_bound_optimal: float
    sq_bound_score: float
    sq_bound_pilot: float
    empirical_mse: float
    coverage: float


ANALYTICS_HEADER = ["instance", "method", "c", "num_blocks", "objective", "sq_bound_optimal", "sq_bound_score",
                    "sq_bound_pilot", "empirical_mse", "coverage"]


def write_analytics_csv(path, rows: Sequence[AnalyticsRow]) -> None:
    """analysis.py:448-470."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(ANALYTICS_HEADER)
        for r in rows:
            w.writerow([r.instance, r.method, r.c, r.num_blocks] +
                       [f"{v:.17g}" for v in (r.objective, r.sq_bound_optimal, r.sq_bound_score,
                                              r.sq_bound_pilot, r.empirical_mse, r.coverage)])
