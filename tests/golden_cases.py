"""Rebuild the seeded inputs behind tests/golden/*.npz (mirrors make_golden.py)."""
import numpy as np


def make_instance(case):
    g = np.random.default_rng(case["seed"])
    M = g.standard_normal((case["m"], case["n"])) * g.lognormal(0, 1.0, case["n"])
    N = g.standard_normal((case["n"], case["p"]))
    if case["zero"]:
        cols, blk = case["zero"]
        M[:, cols] = 0.0
        M[:, blk[0]:blk[1]] = 0.0
    return M, N


def ssm_draws(case):
    return max(1, case["c"] // max(1, int(np.mean(case["sizes"]))))
