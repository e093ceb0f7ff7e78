"""Host side of the numpy-stream reproduction: turning a caller's
``numpy.random.Generator`` into the words the device seeds from, and applying
the caller-visible side effects the reference has on that generator.

Reference behaviour reproduced:
  * ``rng.spawn(K)`` (estimators.py:141, plan.py:456) creates children
    ``SeedSequence(entropy, spawn_key=key + (n_children_spawned + j,))`` and
    advances the parent's ``n_children_spawned`` by K;
  * ``rng.random(count)`` on the caller's own stream (estimators.py:41 via
    sketch_columns, 242 via the SSM baseline) advances its PCG64 state by
    ``count`` steps.
The device side (csrc/rng.cuh) derives each child's PCG64 state itself; the
host only supplies the entropy words and applies the counter/state updates.
"""
from __future__ import annotations

import numpy as np

MASK32 = 0xFFFFFFFF
MASK128 = (1 << 128) - 1
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def _words(v) -> list[int]:
    if isinstance(v, (int, np.integer)):
        v = int(v)
        if v < 0:
            raise ValueError("negative entropy")
        if v == 0:
            return [0]
        out = []
        while v:
            out.append(v & MASK32)
            v >>= 32
        return out
    if isinstance(v, np.ndarray) and v.dtype == np.uint32:
        return [int(x) for x in v.ravel()]
    out: list[int] = []
    for x in v:
        out.extend(_words(x))
    return out


def _pcg64(rng) -> np.random.PCG64:
    bg = rng.bit_generator if isinstance(rng, np.random.Generator) else rng
    if not isinstance(bg, np.random.PCG64):
        raise ValueError("the B200 sampler reproduces numpy PCG64 streams only; "
                         f"got {type(bg).__name__}")
    return bg


def spawn_words(rng, count: int) -> tuple[np.ndarray, int]:
    """Words for ``rng.spawn(count)`` and the index of the first child.

    Applies the side effect (parent's ``n_children_spawned += count``) so later
    calls on ``rng`` see the same state the reference leaves behind.
    """
    bg = _pcg64(rng)
    ss = bg.seed_seq
    if not isinstance(ss, np.random.SeedSequence):
        raise ValueError("generator has no SeedSequence to spawn from")
    if ss.pool_size != 4:
        raise ValueError("only the default SeedSequence pool size (4) is supported")
    run = _words(ss.entropy) if ss.entropy is not None else []
    key = _words(tuple(ss.spawn_key))
    if len(run) < 4:  # children always carry a spawn key, so the run entropy is padded
        run = run + [0] * (4 - len(run))
    first = int(ss.n_children_spawned)
    advance_spawn_counter(ss, count)
    return np.asarray(run + key, dtype=np.uint32), first


def advance_spawn_counter(ss: np.random.SeedSequence, count: int) -> None:
    """``ss.spawn(count)`` for its side effect on the parent (``n_children_spawned += count``,
    which is all the reference's ``rng.spawn(K)`` leaves behind on the caller's generator).

    The public call is the contract; the pickle-state shortcut only skips building ``count``
    child objects and is taken only when the state tuple has the layout this numpy writes
    (entropy, n_children_spawned, pool, pool_size, spawn_key) and the counter reads back as
    expected -- otherwise the parent is put back as it was and ``spawn`` runs."""
    if count <= 0:
        return
    before = ss.n_children_spawned
    st = None
    try:  # (spawn(50) builds 50 child objects, ~0.15 ms: too slow for a 1.1 ms config-2 step)
        st = ss.__reduce__()[2]
        if isinstance(st, tuple) and len(st) == 5 and st[1] == before:
            ss.__setstate_cython__((st[0], before + count, st[2], st[3], st[4]))
            if ss.n_children_spawned == before + count:
                return
            ss.__setstate_cython__(st)
    except Exception:  # numpy internals changed: undo if possible, then the public call
        try:
            if st is not None and ss.n_children_spawned != before:
                ss.__setstate_cython__(st)
        except Exception:
            pass
    if ss.n_children_spawned != before:
        raise RuntimeError("SeedSequence spawn counter could not be restored; refusing to continue")
    ss.spawn(count)


def stream_state(rng) -> np.ndarray:
    """The caller's current PCG64 (state, inc) as 4 uint64 words (hi, lo, hi, lo)."""
    st = _pcg64(rng).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    return np.array([s >> 64, s & ((1 << 64) - 1), inc >> 64, inc & ((1 << 64) - 1)], dtype=np.uint64)


def _jump(state: int, inc: int, delta: int) -> int:
    acc_m, acc_p, cur_m, cur_p = 1, 0, PCG_MULT, inc
    while delta > 0:
        if delta & 1:
            acc_m = (acc_m * cur_m) & MASK128
            acc_p = (acc_p * cur_m + cur_p) & MASK128
        cur_p = ((cur_m + 1) * cur_p) & MASK128
        cur_m = (cur_m * cur_m) & MASK128
        delta >>= 1
    return (acc_m * state + acc_p) & MASK128


def consume(rng, count: int) -> None:
    """Advance the caller's stream as ``rng.random(count)`` would (buffered
    32-bit halves are untouched, exactly like drawing doubles)."""
    bg = _pcg64(rng)
    full = bg.state
    st = full["state"]
    st["state"] = _jump(int(st["state"]), int(st["inc"]), int(count))
    bg.state = full
