"""Multi-GPU approximate product: M's rows and N's columns sharded across ranks.

SURVEY.md §8(e): output tiles of C.D need only the replicated sample (indices,
scales) plus the local M rows / N columns, so the data path has no
communication.  Ranks form a Gr x Gc grid; rank (a, b) = a * Gc + b owns
M[rows_a, :] and N[:, cols_b] and produces CD[rows_a, cols_b].  The exchanges
are small and happen once per call (C1-C3 of the survey):

  C1  the norm pass.  Made EXACT -- every rank ends with the bits a single GPU
      computes, so plans and draws are bit-identical at any GPU count:
      * colsq is NumPy's sequential chain over the rows of M (matrix.py:107-109).
        The columns are split into Gc slabs; rank (a, b) continues the chain of
        column slab b over its rows_a, starting from the accumulator rank
        (a-1, b) handed on (Gr stages, one all-gather each): the chain runs over
        rows 0..m-1 in order, exactly as on one device.
      * rowsq is NumPy's pairwise tree over a row of N (matrix.py:112-114).  The
        column shards cols_b are cut at nodes of that tree (pairwise_shards), so
        rank (a, b) sums complete subtrees for the rows of slab a, and the
        partials are combined in the tree's own order (tree_combine).
      Every byte of M and N is read once across the job.
  C2  K-length partials of the block-product norms g_k^2 (OPL) and of the
      two-step pilot norms over the output tiles: ||X||_F^2 of the whole
      product is the sum of its tiles' (an all-gather and a fixed rank-order
      sum, so every rank holds identical bits whatever algorithm NCCL picks).
  C3  two error scalars (verification only).

Plans, child streams and draws are then computed redundantly on every rank from
identical inputs, so no broadcast is needed.  Grids with Gc not a power of two
(world sizes other than 1, 2, 4, 8, ...) or widths whose tree cannot be cut
into Gc subtrees fall back to balanced column shards and a rank-ordered sum of
row partials (deterministic, equal on all ranks, within rounding of the
single-GPU norms).
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _lib


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


def _pw_split(length: int) -> int:
    """NumPy's pairwise split point (numpy/core/src/umath/loops_utils.h: n2 = n/2, n2 -= n2 % 8)."""
    n2 = length // 2
    return n2 - n2 % 8


def pairwise_shards(p: int, parts: int):
    """Cut [0, p) into `parts` contiguous pieces that are nodes of NumPy's
    pairwise summation tree over a row of width p (parts a power of two and
    every cut node longer than the 128-element leaf), or None if impossible."""
    if parts < 1 or parts & (parts - 1):
        return None
    segs = [(0, p)]
    while len(segs) < parts:
        nxt = []
        for lo, hi in segs:
            if hi - lo <= 128:
                return None
            h = _pw_split(hi - lo)
            nxt += [(lo, lo + h), (lo + h, hi)]
        segs = nxt
    return segs


def tree_combine(parts: list):
    """Combine subtree sums in the pairwise tree's order: ((p0 + p1) + (p2 + p3)) ..."""
    while len(parts) > 1:
        parts = [parts[i] + parts[i + 1] for i in range(0, len(parts), 2)]
    return parts[0]


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
    def exact_rows(self) -> bool:
        """Column shards are pairwise-tree nodes (rowsq combines exactly)."""
        return pairwise_shards(self.p, self.grid[1]) is not None

    def col_shard(self, b: int) -> tuple:
        segs = pairwise_shards(self.p, self.grid[1])
        return segs[b] if segs is not None else shard_range(self.p, self.grid[1], b)

    def row_shard(self, a: int) -> tuple:
        return shard_range(self.m, self.grid[0], a)

    @property
    def rows(self):
        return self.row_shard(self.coords[0])

    @property
    def cols(self):
        return self.col_shard(self.coords[1])

    def colsq_slab(self, b: int) -> tuple:
        """Columns of M whose chains rank (., b) carries (32-column aligned)."""
        units = (self.n + 31) // 32
        lo, hi = shard_range(units, self.grid[1], b)
        return min(self.n, 32 * lo), min(self.n, 32 * hi)

    def rowsq_slab(self, a: int) -> tuple:
        """Rows of N whose partial row sums rank (a, .) computes."""
        return shard_range(self.n, self.grid[0], a)


def _world(group=None) -> int:
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


def _all_gather(buf: torch.Tensor, group=None) -> torch.Tensor:
    """(world, len) gathered copy of every rank's `buf` (gloo: staged through host)."""
    world = _world(group)
    if world == 1 and os.environ.get("BMM_EXCHANGE_WORLD1") != "1":  # (=1: run the collective anyway, tests)
        return buf[None]
    src = buf.contiguous()
    if dist.get_backend(group) == "gloo":  # host collectives: stage device buffers through host memory
        src = src.cpu()
        parts = [torch.empty_like(src) for _ in range(world)]
        dist.all_gather(parts, src, group=group)
        return torch.stack(parts).to(buf.device)
    out = torch.empty((world,) + tuple(src.shape), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src, group=group)
    return out


def exchange_sum(partial: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather `partial` from every rank and sum in rank order (deterministic,
    identical on all ranks)."""
    if _world(group) == 1 and os.environ.get("BMM_EXCHANGE_WORLD1") != "1":
        return partial
    parts = _all_gather(partial, group)
    acc = parts[0].clone()
    for t in parts[1:]:
        acc += t
    return acc


class NcclComm:
    """An NCCL communicator owned by the C-ABI (bmm_nccl_comm_init), for the
    exchanges enqueued on the current stream as C-ABI calls
    (bmm_all_gather_f64_nccl / bmm_exchange_sum_nccl: SURVEY §8(b2) optional
    ncclComm_t variants).  Built over a torch.distributed group, which only
    carries the unique id from rank 0; world 1 needs no group."""

    def __init__(self, group=None):
        import ctypes
        self.world = _world(group)
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        uid = np.zeros(128, dtype=np.uint8)
        if self.rank == 0:
            _lib.call("bmm_nccl_unique_id", uid.ctypes.data)
        if self.world > 1:
            box = [uid.tobytes()]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            uid = np.frombuffer(box[0], dtype=np.uint8).copy()
        ptr = ctypes.c_void_p()
        _lib.call("bmm_nccl_comm_init", ctypes.addressof(ptr), self.world, uid.ctypes.data, self.rank)
        self.comm = ptr.value
        self._ws = None

    def all_gather(self, buf: torch.Tensor) -> torch.Tensor:
        """(world, len) gathered copy of every rank's float64 `buf`."""
        src = buf.contiguous()
        out = torch.empty((self.world,) + tuple(src.shape), dtype=torch.float64, device=src.device)
        _lib.call("bmm_all_gather_f64_nccl", self.comm, src.data_ptr(), src.numel(), out.data_ptr(),
                  _lib.stream_ptr())
        return out

    def exchange_sum(self, buf: torch.Tensor) -> torch.Tensor:
        """The rank-ordered sum of every rank's float64 `buf` (= exchange_sum)."""
        src = buf.contiguous()
        n = src.numel()
        if self._ws is None or self._ws.numel() < self.world * n:
            self._ws = torch.empty(self.world * n, dtype=torch.float64, device=src.device)
        out = torch.empty_like(src)
        _lib.call("bmm_exchange_sum_nccl", self.comm, self.world, src.data_ptr(), n, self._ws.data_ptr(),
                  out.data_ptr(), _lib.stream_ptr())
        return out

    def close(self) -> None:
        if self.comm:
            _lib.call("bmm_nccl_comm_destroy", self.comm)
            self.comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass


def _kernel_colsq(Mslab: torch.Tensor, acc: torch.Tensor, accumulate: bool) -> None:
    rows, cols = Mslab.shape
    if rows == 0 or cols == 0:
        return
    _lib.call("bmm_norms", _lib.matrix_dtype(Mslab), Mslab.data_ptr(), rows, cols, Mslab.stride(0), 0, None, 0, 0,
              0, 1, int(accumulate), acc.data_ptr(), None, _lib.stream_ptr())


def _kernel_rowsq(Nslab: torch.Tensor, out: torch.Tensor) -> None:
    rows, cols = Nslab.shape
    if rows == 0 or cols == 0:
        return
    _lib.call("bmm_norms", _lib.matrix_dtype(Nslab), None, 0, rows, 0, 0, Nslab.data_ptr(), cols, Nslab.stride(0),
              0, 1, 0, None, out.data_ptr(), _lib.stream_ptr())


@dataclass
class ShardExchange:
    """The cross-rank steps of one sharded pipeline (see the module docstring).
    colsq_fn / rowsq_fn are the per-rank norm kernels (the C-ABI by default;
    the CPU tests substitute the oracle's NumPy chains to check the exchange)."""

    layout: ShardLayout
    group: object = None
    colsq_fn: object = field(default=_kernel_colsq)
    rowsq_fn: object = field(default=_kernel_rowsq)
    comm: object = None  # NcclComm: the exchanges as C-ABI calls on its communicator

    def _gather(self, buf: torch.Tensor) -> torch.Tensor:
        if self.comm is not None:
            return self.comm.all_gather(buf)
        return _all_gather(buf, self.group)

    def norms(self, M_local: torch.Tensor, N_local: torch.Tensor, colsq: torch.Tensor, rowsq: torch.Tensor) -> None:
        """Full-length colsq and rowsq (bit-identical to one device when the
        layout is exact) from this rank's M rows and N columns."""
        L = self.layout
        gr, gc = L.grid
        a, b = L.coords
        n = L.n
        dev = colsq.device
        cmax = max(hi - lo for lo, hi in (L.colsq_slab(j) for j in range(gc)))
        rmax = max(hi - lo for lo, hi in (L.rowsq_slab(j) for j in range(gr)))
        buf = torch.zeros(cmax + rmax, dtype=torch.float64, device=dev)
        acc, rpart = buf[:cmax], buf[cmax:]
        r0, r1 = L.rowsq_slab(a)
        self.rowsq_fn(N_local[r0:r1], rpart[:r1 - r0])
        c0, c1 = L.colsq_slab(b)
        gathered0 = None
        for j in range(gr):
            if a == j:
                self.colsq_fn(M_local[:, c0:c1], acc[:c1 - c0], j > 0)
            g = self._gather(buf if j == 0 else acc)
            if j == 0:
                gathered0 = g
            if j + 1 < gr:  # the next row group continues the chains of the same column slab
                acc.copy_(g[(j * gc + b), :cmax])
        for bb in range(gc):
            lo, hi = L.colsq_slab(bb)
            colsq[lo:hi] = g[(gr - 1) * gc + bb, :hi - lo]
        for aa in range(gr):
            lo, hi = L.rowsq_slab(aa)
            parts = [gathered0[aa * gc + bb, cmax:cmax + hi - lo] for bb in range(gc)]
            rowsq[lo:hi] = tree_combine(parts) if L.exact_rows else exchange_sum_list(parts)

    def sum_(self, t: torch.Tensor) -> None:
        """In place: the rank-ordered sum of every rank's partial `t`."""
        if self.comm is not None:
            t.copy_(self.comm.exchange_sum(t))
        else:
            t.copy_(exchange_sum(t, self.group))


def exchange_sum_list(parts: list):
    acc = parts[0].clone()
    for t in parts[1:]:
        acc = acc + t
    return acc


class ShardedApproxProduct:
    """The sharded form of a PipelineGroup over ONE instance: approximate
    products (any of OPL, ONC, UU, ONU, ONMCNR, SSM) of a problem whose M rows
    and N columns are sharded over the process group.  Each member is a
    SketchPipeline of this rank's tile (m_a x n x p_b) whose statistics go
    through a ShardExchange; run() returns this rank's CD[rows_a, cols_b] tile
    for each member.  Buffers are allocated once (construction), the kernels
    are those of the single-GPU pipeline.

    runs: [(method, c)] (SSM: c = number of whole-block draws); c0 for two-step.
    comm: an NcclComm -- the exchanges then run as C-ABI NCCL calls on the
    current stream instead of torch.distributed collectives."""

    def __init__(self, layout: ShardLayout, sizes, runs, *, dtype=torch.float32, c0: int = 0, cap: bool = True,
                 group=None, comm: NcclComm | None = None):
        from .pipeline import PipelineGroup, SketchPipeline
        self.L, self.sizes, self.runs = layout, tuple(int(s) for s in sizes), [(str(mt), int(c)) for mt, c in runs]
        if sum(self.sizes) != layout.n:
            raise ValueError("partition does not cover n")
        self.exchange = ShardExchange(layout, group, comm=comm)
        r0, r1 = layout.rows
        b0, b1 = layout.cols
        self.ma, self.pb = r1 - r0, b1 - b0
        pipes = []
        for meth, c in self.runs:
            if meth == "SSM":
                q = SketchPipeline(self.ma, layout.n, self.pb, self.sizes, 0, "SSM", draws=c, dtype=dtype, cap=cap)
            else:
                q = SketchPipeline(self.ma, layout.n, self.pb, self.sizes, c, meth, dtype=dtype, c0=c0, cap=cap)
            q.exchange = self.exchange
            pipes.append(q)
        self.group = PipelineGroup(pipes, joint=False, shared=len(pipes) > 1)
        self.pipes = pipes

    def run(self, M_local: torch.Tensor, N_local: torch.Tensor, seeds: list) -> list:
        """This rank's tiles CD[rows_a, cols_b], one per run (seeds: one CallSeeds
        per run, identical on every rank)."""
        if tuple(M_local.shape) != (self.ma, self.L.n) or tuple(N_local.shape) != (self.L.n, self.pb):
            raise ValueError("local shards do not match the layout")
        if len(self.pipes) == 1:
            q = self.pipes[0]
            q.set_seeds(seeds[0])
            return [q.launch(M_local, N_local)]
        return self.group.run(M_local, N_local, seeds)

    def check(self) -> None:
        self.group.check()
