"""Multi-GPU approximate product: M's rows and N's columns sharded across ranks.

SURVEY.md §8(e): output tiles of C.D need only the replicated sample (indices,
scales) plus the local M rows / N columns, so the data path has no
communication.  The exchanges are small and happen once per call:

  C1  colsq (n) and rowsq (n) partial sums of squares      -> every rank
  C2  K-length g_k^2 partials (OPL) / pilot^2 partials      -> every rank
  C3  two error scalars (verification only)

Ranks form a Gr x Gc grid; rank (a, b) owns M[rows_a, :] and N[:, cols_b] and
produces CD[rows_a, cols_b].  The norm-pass *work* is split further so each
byte of M and N is read once across the job: rank (a, b) sums squares over
the b-th sub-slab of rows_a (M) and the a-th sub-slab of cols_b (N).

Exchanges are an all-gather of the partials followed by a fixed rank-order
sum, so every rank holds identical bits (identical plans and draws without a
broadcast) and results do not depend on the collective algorithm NCCL picks.
Sharded partial sums change the float64 rounding of colsq/rowsq at the 1e-16
level, so sampled indices match the single-GPU run except with probability
~1e-8 per problem; they are identical across ranks always.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .plan import segsq_engine


def grid_shape(world: int) -> tuple:
    """(Gr, Gc) with Gr * Gc == world, as square as possible, Gc >= Gr."""
    gr = int(np.floor(np.sqrt(world)))
    while world % gr:
        gr -= 1
    return gr, world // gr


def shard_range(total: int, parts: int, idx: int) -> tuple:
    """Balanced contiguous split of range(total) into `parts`; piece `idx`."""
    base, extra = divmod(total, parts)
    lo = idx * base + min(idx, extra)
    return lo, lo + base + (1 if idx < extra else 0)


@dataclass(frozen=True)
class ShardLayout:
    world: int
    rank: int
    m: int
    n: int
    p: int

    @property
    def grid(self):
        return grid_shape(self.world)

    @property
    def coords(self):
        gr, gc = self.grid
        return divmod(self.rank, gc)  # (a, b)

    @property
    def rows(self):
        gr, _ = self.grid
        return shard_range(self.m, gr, self.coords[0])

    @property
    def cols(self):
        _, gc = self.grid
        return shard_range(self.p, gc, self.coords[1])

    @property
    def norm_rows(self):
        """Rows of the local M slab whose squares this rank sums (global row ids)."""
        _, gc = self.grid
        lo, hi = self.rows
        a, b = self.coords
        s0, s1 = shard_range(hi - lo, gc, b)
        return lo + s0, lo + s1

    @property
    def norm_cols(self):
        """Columns of the local N slab whose squares this rank sums (global column ids)."""
        gr, _ = self.grid
        lo, hi = self.cols
        a, b = self.coords
        s0, s1 = shard_range(hi - lo, gr, a)
        return lo + s0, lo + s1


def exchange_sum(partial: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather `partial` from every rank and sum in rank order (deterministic,
    identical on all ranks)."""
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if world == 1:
        return partial
    parts = [torch.empty_like(partial) for _ in range(world)]
    dist.all_gather(parts, partial.contiguous(), group=group)
    acc = parts[0].clone()
    for t in parts[1:]:
        acc += t
    return acc


class ShardedApproxProduct:
    """One approximate product (methods ONC / OPL / UU) of a problem whose M rows
    and N columns are sharded over the process group; returns this rank's
    CD[rows_a, cols_b] tile.  The device steps are the same C-ABI kernels as
    the single-GPU pipeline."""

    def __init__(self, layout: ShardLayout, sizes, c: int, method: str = "ONC", dtype=torch.float32,
                 cap: bool = True, group=None):
        if method not in ("ONC", "OPL", "UU"):
            raise ValueError("sharded path supports ONC, OPL and UU")
        self.L, self.sizes, self.c, self.method, self.cap, self.group = layout, tuple(sizes), int(c), method, cap, group
        self.dtype = dtype
        self.lib = _lib.load()
        dev = _lib.device()
        K, n = len(self.sizes), layout.n
        self.K = K
        off = np.zeros(K + 1, dtype=np.int64)
        np.cumsum(self.sizes, out=off[1:])
        self.offsets = torch.as_tensor(off, device=dev)
        self.sizes_d = torch.as_tensor(np.asarray(self.sizes, np.int64), device=dev)
        f64 = dict(dtype=torch.float64, device=dev)
        i64 = dict(dtype=torch.int64, device=dev)
        self.norms_part = torch.zeros(2 * n, **f64)
        self.probs = torch.empty(n, **f64)
        self.s = torch.empty(K, **f64)
        self.cum = torch.empty(n, **f64)
        self.last = torch.empty(K, **i64)
        self.budgets = torch.empty(K, **i64)
        self.col_off = torch.empty(K + 1, **i64)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.diag = torch.zeros(1, **i64)
        self.c_arr = torch.full((1,), self.c, **i64)
        self.ws_budget = _lib.workspace(self.lib.bmm_budgets_workspace(K))
        self.states = torch.empty(4 * K, **i64)
        W = self.c
        self.column = torch.zeros(W, **i64)
        self.prob = torch.empty(W, **f64)
        self.scale = torch.empty(W, **f64)
        ma = layout.rows[1] - layout.rows[0]
        pb = layout.cols[1] - layout.cols[0]
        self.ma, self.pb = ma, pb
        if method == "UU":
            u = np.concatenate([np.full(nk, 1.0 / nk) for nk in self.sizes])
            self.uprobs = torch.as_tensor(u, device=dev)

    def _c(self, name, *args):
        rc = getattr(self.lib, name)(*args)
        if rc < 0:
            raise RuntimeError(f"{name} failed ({rc}): {self.lib.bmm_last_error().decode()}")

    def run(self, M_local: torch.Tensor, N_local: torch.Tensor, words: np.ndarray, first: int) -> torch.Tensor:
        L, K, n, W = self.L, self.K, self.L.n, self.c
        st = _lib.stream_ptr()
        P = lambda t: t.data_ptr()  # noqa: E731
        dt = _lib.matrix_dtype(M_local)
        r0, r1 = L.rows
        c0, c1 = L.cols
        nr0, nr1 = L.norm_rows
        nc0, nc1 = L.norm_cols
        # C1: partial sums of squares over this rank's share of the bytes
        colsq, rowsq = self.norms_part[:n], self.norms_part[n:]
        colsq.zero_()
        rowsq.zero_()
        Mpart = M_local[nr0 - r0:nr1 - r0]
        Npart = N_local[:, nc0 - c0:nc1 - c0]
        if Mpart.shape[0] > 0:
            self._c("bmm_norms", dt, P(Mpart), Mpart.shape[0], n, M_local.stride(0), 0, None, 0, 0, 0, 1, 0,
                    P(colsq), None, st)
        if Npart.shape[1] > 0:
            self._c("bmm_norms", dt, None, 0, n, 0, 0, Npart.data_ptr(), Npart.shape[1], N_local.stride(0), 0, 1, 0,
                    None, P(rowsq), st)
        full = exchange_sum(self.norms_part, self.group)
        colsq, rowsq = full[:n], full[n:]
        self._c("bmm_block_probs", P(colsq), P(rowsq), n, P(self.offsets), K, 1, max(self.sizes), P(self.probs), P(self.s), None,
                P(self.cum), P(self.last), st)
        aux = None
        if self.method == "OPL":
            # C2: g_k^2 partials of this rank's output tile
            if segsq_engine(max(self.sizes), M_local.shape[0], N_local.shape[1], n) == "i8":
                A, B = M_local.contiguous(), N_local.contiguous()
                if A.dtype != B.dtype:
                    A, B = A.double(), B.double()
                gpart = torch.empty(K, dtype=torch.float64, device=A.device)
                ws = _lib.workspace(self.lib.bmm_segsq_i8_workspace(A.shape[0], B.shape[1], n, K, 1))
                self._c("bmm_segsq_i8", _lib.matrix_dtype(A), P(A), A.stride(0), 0, P(B), B.stride(0), 0,
                        A.shape[0], B.shape[1], n, P(self.offsets), K, 0, 1, P(gpart), P(ws), ws.numel(), st)
            else:
                A = M_local.double() if M_local.dtype != torch.float64 else M_local
                B = N_local.double().contiguous() if N_local.dtype != torch.float64 else N_local.contiguous()
                gpart = torch.empty(K, dtype=torch.float64, device=A.device)
                ws = _lib.workspace(self.lib.bmm_segsq_f64_workspace(A.shape[0], B.shape[1], K, 1))
                self._c("bmm_segsq_f64", P(A), A.stride(0), 0, P(B), B.stride(0), 0, A.shape[0], B.shape[1],
                        P(self.offsets), K, 0, 1, P(gpart), P(ws), ws.numel(), st)
            aux = exchange_sum(gpart, self.group)
        rule = {"ONC": _lib.RULE_ONC, "OPL": _lib.RULE_OPL, "UU": _lib.RULE_UU}[self.method]
        self._c("bmm_budgets", rule, P(self.s) if rule != _lib.RULE_UU else None, P(aux) if aux is not None else None,
                P(self.sizes_d), None, None, K, 1, P(self.c_arr), int(self.cap), P(self.budgets), P(self.col_off),
                P(self.status), P(self.diag), None, P(self.ws_budget), st)
        probs = self.probs
        if self.method == "UU":
            probs = self.uprobs
            self._c("bmm_block_cdf", P(probs), P(self.offsets), K, 1, n, P(self.cum), P(self.last), st)
        words_d = torch.as_tensor(np.ascontiguousarray(words, dtype=np.uint32).view(np.int32), device=M_local.device)
        first_d = torch.as_tensor(np.array([first], dtype=np.int64), device=M_local.device)
        self._c("bmm_seed_streams", P(words_d), len(words), P(first_d), K, 1, P(self.states), st)
        self._c("bmm_sample", P(probs), P(self.cum), P(self.last), P(self.offsets), K, 1, n, max(self.sizes),
                P(self.budgets), P(self.col_off), W, P(self.states), P(self.column), P(self.prob), P(self.scale), st)
        ma, pb = self.ma, self.pb
        # compressed sketch (one term per distinct drawn column), as SketchPipeline
        dev = M_local.device
        kcol = torch.empty(W, dtype=torch.int64, device=dev)
        ksc = torch.empty(W, dtype=torch.float64, device=dev)
        kcnt = torch.empty(1, dtype=torch.int64, device=dev)
        wsc = _lib.workspace(self.lib.bmm_compress_workspace(n, 1))
        self._c("bmm_compress_sketch", P(self.column), P(self.scale), W, W, n, 1, P(wsc), wsc.numel(), P(kcol),
                P(ksc), P(kcnt), st)
        if M_local.dtype == torch.float32 and W % 8 == 0:
            a_hi = torch.empty(ma * W, dtype=torch.float32, device=dev)
            a_x = torch.empty_like(a_hi)
            b_hi = torch.empty(pb * W, dtype=torch.float32, device=dev)
            b_x = torch.empty_like(b_hi)
            Nc = N_local.contiguous()
            self._c("bmm_gather_f32split_dk", dt, P(M_local), M_local.stride(0), 0, P(Nc), Nc.stride(0), 0, ma, pb,
                    P(kcol), P(ksc), W, W, P(kcnt), 1, P(a_hi), P(a_x), P(b_hi), P(b_x), st)
            out = torch.empty((ma, pb), dtype=torch.float32, device=dev)
            self._c("bmm_gemm_f32split_dk", P(a_hi), P(a_x), P(b_hi), P(b_x), ma, pb, W, P(kcnt), 1, P(out), pb, 0,
                    st)
            return out
        C = torch.empty((ma, W), dtype=torch.float64, device=dev)
        D = torch.empty((W, pb), dtype=torch.float64, device=dev)
        self._c("bmm_gather_dk", dt, _lib.BMM_F64, P(M_local), M_local.stride(0), 0, P(N_local), N_local.stride(0),
                0, ma, pb, P(kcol), P(ksc), W, W, P(kcnt), 1, P(C), W, 0, P(D), pb, 0, st)
        out = torch.empty((ma, pb), dtype=torch.float64, device=dev)
        ws = _lib.workspace(self.lib.bmm_gemm_f64_workspace(ma, pb, W, 1))
        self._c("bmm_gemm_f64_dk", P(C), W, 0, P(D), pb, 0, ma, pb, W, P(kcnt), 1, P(out), pb, 0, P(ws), ws.numel(),
                st)
        return out

    def check(self):
        from .plan import raise_status
        raise_status(int(self.status.item()), int(self.diag.item()), self.c)
