"""CPU oracle: a NumPy restatement of the reference hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): used by tests/ as the
parity checker, by __graft_entry__.smoke(), and as the timed CPU baseline in
bench.py (``cpu_baseline`` / ``--impl reference``, kind "port").  The product
package never imports it.

It restates, as plain functions over arrays, the reference package
``blockmm`` (pkg/src/blockmm, pure Python/NumPy, numpy>=1.25 / scipy>=1.10):

  norms            matrix.py:107-114      np.linalg.norm(M, axis=0) / (N, axis=1)
  index scores     plan.py:165-167        column_norms * row_norms
  score sums       plan.py:170-173        np.add.reduceat over block starts
  probabilities    plan.py:192-206        p = s/sum(s); p/sum(p); zero block -> 0
  block products   plan.py:176-189        ||M^k @ N_k||_F  (BLAS)
  integerize       plan.py:242-347        largest remainder, caps, floors, fixpoint
  size weights     plan.py:350-361,465    sqrt(max(s^2-g^2,0)); sqrt(|s^2-pilot^2|)
  caps             plan.py:373-380
  allocators       plan.py:383-480
  SSM weights      plan.py:483-496
  draws            estimators.py:34-44    cumsum, searchsorted(right), clamp
  sketch           estimators.py:55-81
  estimate         estimators.py:125-175
  two-step         estimators.py:185-210
  SSM estimate     estimators.py:221-253
  relative error   analysis.py:318-325
  replications     analysis.py:343-366,390-416   (Monte Carlo, §8 f1)
  variance         analysis.py:57-116            (exact analytics, §8 f2)

Randomness uses numpy's own Generator/PCG64 -- the reference's third-party
dependency -- so streams are the reference's by construction; the restated
stream algorithms live in oracle/numpy_rng.py.

Pinning: tests/test_oracle_golden.py checks this module against golden
vectors produced by running the reference itself in the build container
(tests/golden/make_golden.py), bit-exact for indices/budgets/probabilities
and to BLAS rounding for products.

Difference from the reference, by design: the reference recomputes the norm
pass 2-3 times per allocator (plan.py:165-173 via optimal_probabilities,
score_sums and block_scores); this port computes it once.  As a CPU baseline
it is therefore somewhat faster than the reference itself (conservative).
"""
from __future__ import annotations

import numpy as np

RADICAND_SLACK = 1e-9


# ---------------------------------------------------------------- norms / scores

def colsq(M: np.ndarray) -> np.ndarray:
    """Sum of squares per column, NumPy order (sequential over rows for C order)."""
    return np.add.reduce(M * M, axis=0)


def rowsq(N: np.ndarray) -> np.ndarray:
    """Sum of squares per row, NumPy pairwise order along the contiguous axis."""
    return np.add.reduce(N * N, axis=1)


def colsq_chunked(M: np.ndarray, rows: int = 4096) -> np.ndarray:
    """colsq of a (possibly float32) matrix in float64 with bounded memory.

    The chain continues across row slabs, so the result equals colsq on the
    whole float64-upcast matrix bit for bit."""
    acc = None
    for r0 in range(0, M.shape[0], rows):
        sl = np.asarray(M[r0:r0 + rows], dtype=np.float64)
        sq = sl * sl
        if acc is not None:
            sq = np.concatenate([acc[None, :], sq], axis=0)
        acc = np.add.reduce(sq, axis=0)
    return acc if acc is not None else np.zeros(M.shape[1])


def rowsq_chunked(N: np.ndarray, rows: int = 4096) -> np.ndarray:
    out = np.empty(N.shape[0])
    for r0 in range(0, N.shape[0], rows):
        sl = np.asarray(N[r0:r0 + rows], dtype=np.float64)
        out[r0:r0 + rows] = np.add.reduce(sl * sl, axis=1)
    return out


def offsets_of(sizes) -> np.ndarray:
    return np.concatenate(([0], np.cumsum(np.asarray(sizes, dtype=np.int64))))


def block_stats(cs: np.ndarray, rs: np.ndarray, sizes):
    """(flat optimal probabilities, score sums s_k) from the squared norms."""
    sc = np.sqrt(cs) * np.sqrt(rs)
    off = offsets_of(sizes)
    s = np.add.reduceat(sc, off[:-1])
    probs = np.empty_like(sc)
    for k in range(len(sizes)):
        seg = sc[off[k]:off[k + 1]]
        tot = seg.sum()
        if tot == 0.0:
            probs[off[k]:off[k + 1]] = 0.0
        else:
            q = seg / tot
            probs[off[k]:off[k + 1]] = q / q.sum()
    return probs, s


def block_product_sq(M: np.ndarray, N: np.ndarray, sizes) -> np.ndarray:
    """||M^k @ N_k||_F^2 per block (BLAS order; tolerance-level reference)."""
    off = offsets_of(sizes)
    out = np.empty(len(sizes))
    for k in range(len(sizes)):
        P = M[:, off[k]:off[k + 1]] @ N[off[k]:off[k + 1], :]
        f = P.ravel()
        out[k] = float(np.sqrt(f @ f)) ** 2
    return out


def block_norm_weights(cs: np.ndarray, rs: np.ndarray, sizes) -> np.ndarray:
    """||M^k||_F * ||N_k||_F (SSM, Eq. 1.4) from the squared column/row norms."""
    off = offsets_of(sizes)
    return np.array([np.sqrt(cs[off[k]:off[k + 1]].sum()) * np.sqrt(rs[off[k]:off[k + 1]].sum())
                     for k in range(len(sizes))])


# ---------------------------------------------------------------- integer budgets

class OracleAssert(AssertionError):
    pass


def integerize(w, c: int, caps=None, floors=None) -> np.ndarray:
    """Largest remainder with floors and caps, iterated to a fixpoint.

    Cap pins are permanent; floor pins are recomputed whenever a new cap pin
    appears; leftovers with zero weight get the remaining budget in index
    order; remainders are ranked descending with ties in index order."""
    w = np.asarray(w, dtype=np.float64)
    if w.ndim != 1 or w.size == 0:
        raise ValueError("weights must be a nonempty vector")
    if not np.isfinite(w).all() or (w < 0).any():
        raise ValueError("weights must be finite and >= 0")
    if w.sum() == 0.0:
        raise ValueError("all weights are zero")
    c = int(c)
    if c < 0:
        raise ValueError("budget must be >= 0")
    K = w.size
    lo = (w > 0 if floors is None else np.asarray(floors, dtype=bool)).astype(np.int64)
    hi = np.full(K, c, np.int64) if caps is None else np.minimum(np.asarray(caps, np.int64), c)
    if (hi < lo).any():
        raise ValueError("some cap lies below the required floor of 1")
    if lo.sum() > c:
        raise ValueError(f"budget c={c} is below the {int(lo.sum())} required floors")
    if hi.sum() < c:
        raise ValueError(f"budget c={c} exceeds the total caps {int(hi.sum())}")

    at_cap = np.zeros(K, bool)
    for _ in range(K + 1):
        at_floor = np.zeros(K, bool)
        restart = False
        while not restart:
            free = np.flatnonzero(~at_cap & ~at_floor)
            left = c - int(hi[at_cap].sum()) - int(lo[at_floor].sum())
            result = np.where(at_cap, hi, np.where(at_floor, lo, 0))
            if free.size == 0:
                if left != 0:
                    raise OracleAssert("apportionment did not converge")
                return result
            wf = w[free]
            tot = wf.sum()
            if tot == 0.0:
                for i in free:
                    give = min(left, int(hi[i]))
                    result[i] = give
                    left -= give
                if left != 0:
                    raise OracleAssert("apportionment did not converge")
                return result
            share = left * wf / tot
            over = share > hi[free] + 1e-12
            if over.any():
                at_cap[free[over]] = True
                restart = True
                continue
            under = share < lo[free]
            if under.any():
                at_floor[free[under]] = True
                continue
            base = np.floor(share).astype(np.int64)
            short = left - int(base.sum())
            rank = np.argsort(-(share - base), kind="stable")
            for j in rank:
                if short == 0:
                    break
                if base[j] < hi[free[j]]:
                    base[j] += 1
                    short -= 1
            if short != 0:
                raise OracleAssert("apportionment failed to place the full budget")
            result[free] = base
            return result
    raise OracleAssert("apportionment did not converge")


def caps_for(sizes, cap: bool, c: int, s=None) -> np.ndarray:
    out = np.asarray(sizes, np.int64).copy() if cap else np.full(len(sizes), int(c), np.int64)
    if s is not None:
        out = np.where(s > 0, out, 0).astype(np.int64)
    return out


def plan_budgets(rule: str, sizes, c: int, s=None, aux_sq=None, cap: bool = True):
    """Budgets (and fallback note flag) for rule in {ONC, OPL, TWO_STEP, UU}.

    aux_sq: g_k^2 for OPL, pilot_k^2 for TWO_STEP."""
    if rule == "UU":
        K = len(sizes)
        return integerize(np.ones(K), c, caps=caps_for(sizes, cap, c), floors=np.ones(K, bool)), False
    if s.sum() == 0.0:
        raise ValueError("all blocks have zero score: nothing to sample")
    note = False
    if rule == "ONC":
        w = s
    elif rule == "OPL":
        g = np.sqrt(aux_sq)
        if (g > s * (1 + RADICAND_SLACK) + 1e-300).any():
            raise ValueError("exact product norm exceeds score sum (Cauchy-Schwarz violated)")
        rad = s ** 2 - g ** 2
        if (rad < -RADICAND_SLACK * s ** 2).any():
            raise ValueError("radicand negative beyond rounding slack")
        w = np.sqrt(np.maximum(rad, 0.0))
    elif rule == "TWO_STEP":
        pn = np.sqrt(aux_sq)
        w = np.sqrt(np.abs(s ** 2 - pn ** 2))
    else:
        raise ValueError(rule)
    if rule in ("OPL", "TWO_STEP") and w.sum() == 0.0:
        w, note = s, True
    budgets = integerize(w, c, caps=caps_for(sizes, cap, c, s), floors=s > 0)
    # SamplingPlan.__post_init__ (plan.py:146-152): the zero-weight hand-out
    # (plan.py:311-322) ignores floors, so a scored block can end at 0
    for k in range(len(sizes)):
        if (budgets[k] == 0) != (not s[k] > 0):
            raise ValueError(f"block {k}: zero budget and zero-probability flag must coincide")
    return budgets, note


# ---------------------------------------------------------------- sampling

def draw(p: np.ndarray, count: int, gen: np.random.Generator) -> np.ndarray:
    """Inverse-CDF draws, never returning a zero-probability index."""
    cdf = np.cumsum(p)
    nz = np.flatnonzero(p > 0)
    if nz.size == 0:
        raise ValueError("probability vector has empty support")
    u = gen.random(count)
    return np.minimum(np.searchsorted(cdf, u, side="right"), nz[-1])


def sketch(M, N, sizes, probs_flat, budgets, streams):
    """Per-block draws on the given streams; returns the flat draw log and C, D."""
    off = offsets_of(sizes)
    cols, prob, scale = [], [], []
    for k, ck in enumerate(budgets):
        ck = int(ck)
        if ck == 0:
            continue
        p = probs_flat[off[k]:off[k + 1]]
        idx = draw(p, ck, streams[k])
        pk = p[idx]
        cols.append(off[k] + idx)
        prob.append(pk)
        scale.append(1.0 / np.sqrt(ck * pk))
    if cols:
        cols, prob, scale = np.concatenate(cols), np.concatenate(prob), np.concatenate(scale)
    else:
        cols, prob, scale = np.zeros(0, np.int64), np.zeros(0), np.zeros(0)
    C = M[:, cols] * scale
    D = N[cols, :] * scale[:, None]
    return cols.astype(np.int64), prob, scale, C, D


def instance_stats(M, N, sizes):
    cs, rs = colsq(M), rowsq(N)
    probs, s = block_stats(cs, rs, sizes)
    return cs, rs, probs, s


def two_step_pilot(M, N, sizes, c0: int, method: str, rng: np.random.Generator, probs=None, s=None):
    """Pilot half of estimate_product_two_step (estimators.py:201-208 spawn,
    plan.py:448-464 pilot): returns (pilot_sq, pilot columns, pilot scales,
    main generator).  pilot_sq_k = ||C0_k D0_k||_F^2 in BLAS order."""
    sizes = list(sizes)
    K = len(sizes)
    if probs is None or s is None:
        _, _, probs, s = instance_stats(M, N, sizes)
    p0 = np.concatenate([np.full(nk, 1.0 / nk) for nk in sizes]) if method == "ONU" else probs
    pilot_rng, main_rng = rng.spawn(2)
    pc = int(c0) // K
    if pc < 1:
        raise ValueError(f"c0={c0} gives no pilot draws for K={K} blocks")
    off = offsets_of(sizes)
    live = np.array([p0[off[k]:off[k + 1]].sum() != 0.0 for k in range(K)])
    if s.sum() == 0.0:
        raise ValueError("all blocks have zero score: nothing to sample")
    pstreams = pilot_rng.spawn(K)
    pbud = np.where(live, pc, 0)
    pcols, _, pscale, C0, D0 = sketch(M, N, sizes, p0, pbud, pstreams)
    pilot_sq = np.zeros(K)
    po = offsets_of(pbud)
    for k in range(K):
        if pbud[k]:
            P = C0[:, po[k]:po[k + 1]] @ D0[po[k]:po[k + 1], :]
            f = P.ravel()
            pilot_sq[k] = float(np.sqrt(f @ f)) ** 2
    return pilot_sq, pcols, pscale, main_rng


def approx_product(M, N, sizes, c: int, method: str, rng: np.random.Generator, c0: int = 0,
                   cap: bool = True, keep_sketch: bool = False) -> dict:
    """One approximate product through the reference composition:
    allocate_{optimal,by_score_sums,uniform} + estimate_product, or
    estimate_product_two_step for ONU / ONMCNR."""
    sizes = list(sizes)
    K = len(sizes)
    out: dict = {"method": method}
    cs, rs, probs, s = instance_stats(M, N, sizes)
    if method in ("ONU", "ONMCNR"):
        pilot_sq, pcols, pscale, main_rng = two_step_pilot(M, N, sizes, c0, method, rng, probs, s)
        budgets, note = plan_budgets("TWO_STEP", sizes, c, s=s, aux_sq=pilot_sq, cap=cap)
        out.update(pilot_sq=pilot_sq, pilot_columns=pcols, pilot_scale=pscale)
        stream_rng = main_rng
    else:
        if method == "UU":
            probs = np.concatenate([np.full(nk, 1.0 / nk) for nk in sizes])
            budgets, note = plan_budgets("UU", sizes, c, cap=cap)
        elif method == "ONC":
            budgets, note = plan_budgets("ONC", sizes, c, s=s, cap=cap)
        elif method == "OPL":
            gsq = block_product_sq(M, N, sizes)
            budgets, note = plan_budgets("OPL", sizes, c, s=s, aux_sq=gsq, cap=cap)
            out["gsq"] = gsq
        else:
            raise ValueError(method)
        stream_rng = rng
    streams = stream_rng.spawn(K)
    cols, prob, scale, C, D = sketch(M, N, sizes, probs, budgets, streams)
    out.update(colsq=cs, rowsq=rs, probs=probs, s=s, budgets=budgets, note=note,
               columns=cols, prob=prob, scale=scale, CD=C @ D)
    if keep_sketch:
        out.update(C=C, D=D)
    return out


def ssm_product(M, N, sizes, draws: int, rng: np.random.Generator, q=None) -> dict:
    """Whole-block baseline: q_k ∝ ||M^k||_F ||N_k||_F, draws from the caller stream."""
    off = offsets_of(sizes)
    if q is None:
        f = np.array([np.linalg.norm(M[:, off[k]:off[k + 1]]) * np.linalg.norm(N[off[k]:off[k + 1], :])
                      for k in range(len(sizes))])
        if f.sum() == 0.0:
            raise ValueError("all blocks have zero norm: nothing to sample")
        q = f / f.sum()
    idx = draw(q, int(draws), rng)
    sc = 1.0 / np.sqrt(int(draws) * q[idx])
    C = np.hstack([sc[t] * M[:, off[k]:off[k + 1]] for t, k in enumerate(idx)])
    D = np.vstack([sc[t] * N[off[k]:off[k + 1], :] for t, k in enumerate(idx)])
    return {"q": q, "blocks": idx.astype(np.int64), "prob": q[idx], "scale": sc, "CD": C @ D}


def frob_errors(exact: np.ndarray, approx: np.ndarray) -> tuple:
    """(||exact-approx||_F^2, ||exact||_F^2)."""
    d = (exact - approx).ravel()
    e = exact.ravel()
    return float(d @ d), float(e @ e)


# ---------------------------------------------------------------- §8(f): Monte Carlo and analytics

def replicate(M, N, sizes, probs_flat, budgets, rng: np.random.Generator, reps: int, entry=None) -> dict:
    """``reps`` replications of estimate_product under one plan on
    ``rng.spawn(reps)`` (analysis.py:359-362, 412-413): per replication the
    drawn columns, ||CD - MN||_F^2 (reference: frobenius_norm(...)**2) and
    optionally CD[entry]."""
    K = len(sizes)
    exact = M @ N
    cols, sq, ent = [], [], []
    for stream in rng.spawn(reps):
        c, _, _, C, D = sketch(M, N, sizes, probs_flat, budgets, stream.spawn(K))
        CD = C @ D
        d = (CD - exact).ravel()
        sq.append(float(np.sqrt(d @ d)) ** 2)
        cols.append(c)
        if entry is not None:
            ent.append(CD[entry])
    return {"columns": np.array(cols), "sq_error": np.array(sq), "entry": np.array(ent)}


def elementwise_variance(M, N, sizes, probs_flat, budgets) -> np.ndarray:
    """analysis.py:57-90 (validation errors included)."""
    off = offsets_of(sizes)
    b = np.asarray(budgets, dtype=np.float64)
    var = np.zeros((M.shape[0], N.shape[1]))
    for k in range(len(sizes)):
        Mk, Nk = M[:, off[k]:off[k + 1]], N[off[k]:off[k + 1]]
        p = probs_flat[off[k]:off[k + 1]]
        contrib = np.sqrt((Mk * Mk).sum(axis=0)) * np.sqrt((Nk * Nk).sum(axis=1))
        pos = p > 0
        if (contrib[~pos] > 0).any():
            raise ValueError(f"block {k}: zero probability at a contributing column")
        exact_sq = (Mk @ Nk) ** 2
        term1 = (Mk[:, pos] ** 2 / p[pos]) @ (Nk[pos, :] ** 2)
        num = term1 - exact_sq
        if b[k] == 0:
            if np.abs(num).max(initial=0.0) > 1e-12 * max(1.0, float(term1.max(initial=0.0))):
                raise ValueError(f"block {k}: zero budget on a block with sampling variance")
            continue
        var += num / b[k]
    return var


def expected_sq_error(M, N, sizes, probs_flat, budgets) -> float:
    """analysis.py:93-116."""
    off = offsets_of(sizes)
    b = np.asarray(budgets, dtype=np.float64)
    total = 0.0
    for k in range(len(sizes)):
        Mk, Nk = M[:, off[k]:off[k + 1]], N[off[k]:off[k + 1]]
        p = probs_flat[off[k]:off[k + 1]]
        contrib = np.linalg.norm(Mk, axis=0) * np.linalg.norm(Nk, axis=1)
        pos = p > 0
        if (contrib[~pos] > 0).any():
            raise ValueError(f"block {k}: zero probability at a contributing column")
        term1 = float((contrib[pos] ** 2 / p[pos]).sum())
        num = term1 - float(((Mk @ Nk) ** 2).sum())
        if b[k] == 0:
            if abs(num) > 1e-12 * max(1.0, term1):
                raise ValueError(f"block {k}: zero budget on a block with sampling variance")
            continue
        total += num / b[k]
    return total
