"""Seeded synthetic instances for the five BASELINE.json configs.

The paper's experiments and BASELINE.json's configs are synthetic; these
generators follow SURVEY.md §8(d) (seed root 210504940, data stream
SeedSequence(ROOT, spawn_key=(cfg, 0)), sampling stream
SeedSequence(ROOT, spawn_key=(cfg, 1, rep))).  Shared by bench.py and the
tests; not part of the product package.

cfg1  M 200x10000, N 10000x200 fp64 N(0,1); K=100 x 100; W = 2000 (c=20 blocks)
cfg2  500x20000 / 20000x500 fp64, N(0,1) x lognormal(0,1.5) per column of M /
      row of N; K=50 unequal blocks (>=100); c in {10,20,40} -> W in {4k,8k,16k}
cfg3  1000x100000 / 100000x1000 fp64 Student-t(2); K=1000 x 100; two-step,
      pilot 5/block (c0_col = 5000), W = 20000 (c=200 blocks)
cfg4  16384x262144 / 262144x16384 fp32 N(0,1) x per-block U[0.1,10] (independent
      for M^k and N_k); K=4096 x 64; W = 32768 (c=512 blocks)
cfg5  4096 x (256x4096 / 4096x256) fp32 N(0,1) x lognormal(0,1) per column / row;
      K=64 x 64; W = 1024 (c=16 blocks) per problem
"""
from __future__ import annotations

import numpy as np

ROOT = 210504940

CONFIGS = {
    "cfg1": dict(m=200, n=10000, p=200, K=100, W=2000, dtype="f64"),
    "cfg2": dict(m=500, n=20000, p=500, K=50, W=(4000, 8000, 16000), dtype="f64", c0=500),
    "cfg3": dict(m=1000, n=100000, p=1000, K=1000, W=20000, dtype="f64", c0=5000),
    "cfg4": dict(m=16384, n=262144, p=16384, K=4096, W=32768, dtype="f32"),
    "cfg5": dict(batch=4096, m=256, n=4096, p=256, K=64, W=1024, dtype="f32"),
}


def data_rng(cfg: int, *extra) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(ROOT, spawn_key=(cfg, 0) + tuple(extra)))


def sample_rng(cfg: int, rep: int = 0, *extra) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(ROOT, spawn_key=(cfg, 1, rep) + tuple(extra)))


def cfg1(scale: int = 1):
    g = data_rng(1)
    m, n, p = 200, 10000 // scale, 200
    M = g.standard_normal((m, n))
    N = g.standard_normal((n, p))
    sizes = (100,) * (n // 100)
    return M, N, sizes


def cfg2_sizes(g: np.random.Generator, n: int = 20000, K: int = 50, floor: int = 100) -> tuple:
    cuts = np.sort(g.choice(np.arange(1, n - K * floor), K - 1, replace=False))
    sizes = floor + np.diff(np.concatenate(([0], cuts, [n - K * floor])))
    return tuple(int(s) for s in sizes)


def cfg2(n: int = 20000, m: int = 500, p: int = 500, K: int = 50):
    g = data_rng(2)
    sizes = cfg2_sizes(g, n, K, 100 if n >= 100 * K * 2 else max(1, n // (2 * K)))
    a = g.lognormal(0.0, 1.5, n)
    b = g.lognormal(0.0, 1.5, n)
    M = g.standard_normal((m, n)) * a
    N = g.standard_normal((n, p)) * b[:, None]
    return M, N, sizes


def cfg3(m: int = 1000, n: int = 100000, p: int = 1000, K: int = 1000):
    g = data_rng(3)
    M = g.standard_t(2, (m, n))
    N = g.standard_t(2, (n, p))
    return M, N, (n // K,) * K


def cfg5_problem(b: int, m: int = 256, n: int = 4096, p: int = 256):
    """Problem b of the batched config (float32)."""
    g = data_rng(5, b)
    M = (g.standard_normal((m, n), dtype=np.float32) * g.lognormal(0.0, 1.0, n).astype(np.float32))
    N = (g.standard_normal((n, p), dtype=np.float32) * g.lognormal(0.0, 1.0, n).astype(np.float32)[:, None])
    return M.astype(np.float32), N.astype(np.float32)


def cfg4_scales(K: int = 4096):
    g = data_rng(4)
    return g.uniform(0.1, 10.0, K), g.uniform(0.1, 10.0, K)
