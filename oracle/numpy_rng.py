"""Restatement of numpy's SeedSequence / PCG64 / Generator.random streams.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The reference draws every uniform through ``numpy.random.Generator`` built on
PCG64 (third-party dependency ``numpy>=1.25``, ``pkg/pyproject.toml:10-13``;
this image pins numpy 2.3.5).  Call sites on the hot path:

* ``rng.spawn(K)``           -- ``pkg/src/blockmm/estimators.py:141``
* ``rng.spawn(2)``           -- ``pkg/src/blockmm/estimators.py:207``
* ``rng.spawn(K)`` (pilot)   -- ``pkg/src/blockmm/plan.py:456``
* ``rng.random(count)``      -- ``pkg/src/blockmm/estimators.py:41``

numpy ships no ``.pyx`` sources here, so this module restates the published
algorithms (M.E. O'Neill's seed_seq hashing as adopted by numpy's
``SeedSequence`` with pool size 4; PCG XSL-RR 128/64 with the "set-seq"
seeding; 53-bit doubles ``(next64 >> 11) * 2**-53``).  The restatement is
pinned against live numpy known-answer vectors in ``tests/test_oracle_rng.py``
and ``tests/golden/rng_kat.json``.  The device sampler
(``paper_2105_04940_b200/csrc/rng.cuh``) implements the same arithmetic.
"""
from __future__ import annotations

MASK32 = 0xFFFFFFFF
MASK64 = 0xFFFFFFFFFFFFFFFF
MASK128 = (1 << 128) - 1

INIT_A = 0x43B0D7E5
MULT_A = 0x931E8875
INIT_B = 0x8B51F9DD
MULT_B = 0x58F38DED
MIX_MULT_L = 0xCA01F9DD
MIX_MULT_R = 0x4973F715
XSHIFT = 16
POOL_SIZE = 4

PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def int_to_words(v: int) -> list[int]:
    """Little-endian 32-bit words of a non-negative int (0 -> [0])."""
    if v < 0:
        raise ValueError("negative entropy")
    if v == 0:
        return [0]
    out = []
    while v:
        out.append(v & MASK32)
        v >>= 32
    return out


def coerce_words(x) -> list[int]:
    """Entropy / spawn-key coercion to a flat uint32 word list."""
    if isinstance(x, int):
        return int_to_words(x)
    words: list[int] = []
    for v in x:
        words.extend(coerce_words(int(v)) if not isinstance(v, (list, tuple)) else coerce_words(v))
    return words


def assembled_entropy(entropy, spawn_key) -> list[int]:
    run = coerce_words(entropy) if entropy is not None else []
    spawn = coerce_words(tuple(spawn_key))
    if spawn and len(run) < POOL_SIZE:
        run = run + [0] * (POOL_SIZE - len(run))
    return run + spawn


def _hashmix(value: int, hc: list[int]) -> int:
    value = (value ^ hc[0]) & MASK32
    hc[0] = (hc[0] * MULT_A) & MASK32
    value = (value * hc[0]) & MASK32
    value ^= value >> XSHIFT
    return value


def _mix(x: int, y: int) -> int:
    r = (MIX_MULT_L * x - MIX_MULT_R * y) & MASK32
    r ^= r >> XSHIFT
    return r


def seed_pool(entropy, spawn_key) -> list[int]:
    """The 4-word mixed pool of ``SeedSequence(entropy, spawn_key=...)``."""
    ent = assembled_entropy(entropy, spawn_key)
    hc = [INIT_A]
    pool = [_hashmix(ent[i] if i < len(ent) else 0, hc) for i in range(POOL_SIZE)]
    for i_src in range(POOL_SIZE):
        for i_dst in range(POOL_SIZE):
            if i_src != i_dst:
                pool[i_dst] = _mix(pool[i_dst], _hashmix(pool[i_src], hc))
    for i_src in range(POOL_SIZE, len(ent)):
        for i_dst in range(POOL_SIZE):
            pool[i_dst] = _mix(pool[i_dst], _hashmix(ent[i_src], hc))
    return pool


def generate_state_u32(pool: list[int], n_words32: int) -> list[int]:
    hc = INIT_B
    out = []
    for i in range(n_words32):
        v = pool[i % POOL_SIZE]
        v ^= hc
        hc = (hc * MULT_B) & MASK32
        v = (v * hc) & MASK32
        v ^= v >> XSHIFT
        out.append(v)
    return out


def generate_state_u64(pool: list[int], n_words64: int) -> list[int]:
    w = generate_state_u32(pool, 2 * n_words64)
    return [w[2 * i] | (w[2 * i + 1] << 32) for i in range(n_words64)]


class PCG64:
    """PCG XSL-RR 128/64 with numpy's set-seq seeding from a SeedSequence."""

    def __init__(self, entropy, spawn_key=()):
        s = generate_state_u64(seed_pool(entropy, spawn_key), 4)
        initstate = (s[0] << 64) | s[1]
        initseq = (s[2] << 64) | s[3]
        self.inc = ((initseq << 1) | 1) & MASK128
        self.state = 0
        self._step()
        self.state = (self.state + initstate) & MASK128
        self._step()

    def _step(self):
        self.state = (self.state * PCG_MULT + self.inc) & MASK128

    def next64(self) -> int:
        self._step()
        st = self.state
        rot = st >> 122
        x = ((st >> 64) ^ st) & MASK64
        return ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64

    def random(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)


def child_stream(entropy, parent_key, child_index) -> PCG64:
    """Stream k of ``Generator.spawn``: key = parent_key + (child_index,)."""
    return PCG64(entropy, tuple(parent_key) + (int(child_index),))


def pool_from_assembled(ent: list[int]) -> list[int]:
    """seed_pool for an already-assembled uint32 entropy list (device input layout)."""
    hc = [INIT_A]
    pool = [_hashmix(ent[i] if i < len(ent) else 0, hc) for i in range(POOL_SIZE)]
    for i_src in range(POOL_SIZE):
        for i_dst in range(POOL_SIZE):
            if i_src != i_dst:
                pool[i_dst] = _mix(pool[i_dst], _hashmix(pool[i_src], hc))
    for i_src in range(POOL_SIZE, len(ent)):
        for i_dst in range(POOL_SIZE):
            pool[i_dst] = _mix(pool[i_dst], _hashmix(ent[i_src], hc))
    return pool
