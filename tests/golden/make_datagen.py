"""Golden instances of the reference's generators (
pkg/src/blockmm/datagen.py:55-110) for the numpy-stream mode of
paper_2105_04940_b200.datagen: M, N and the next raw 64-bit word of the caller's
generator after each call (its state must advance exactly as in the reference).

Runs the REFERENCE package (``blockmm`` from /root/reference/pkg/src), so it
only works in the build container; the .npz output is committed.  Re-run with

    python tests/golden/make_datagen.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from blockmm import datagen as rd  # noqa: E402  (the reference, read-only)

# (name, heavy, m, n, p, seed, left (scale, rho) or None, right or None, location)
CASES = [
    ("normal_default", False, 7, 50, 5, 3, None, None, None),
    ("normal_specs", False, 33, 301, 65, 11, (1.5, 0.6), (2.0, -0.4), None),
    ("normal_vec", False, 1, 9, 1, 5, (0.3, 0.0), (4.0, 0.95), None),
    ("heavy_ones", True, 7, 50, 5, 3, None, None, "ones"),
    ("heavy_zero", True, 40, 257, 31, 12, (1.0, -0.8), (0.5, 0.3), "zero"),
]


def main():
    out = {}
    for name, heavy, m, n, p, seed, left, right, loc in CASES:
        rng = np.random.default_rng(seed)
        cl = rd.CovarianceSpec(m, *left) if left else None
        cr = rd.CovarianceSpec(p, *right) if right else None
        if heavy:
            M, N = rd.gen_heavy_tail_instance(m, n, p, rng, cl, cr, location=loc)
        else:
            M, N = rd.gen_normal_instance(m, n, p, rng, cl, cr)
        out[name + "_M"] = M
        out[name + "_N"] = N
        out[name + "_next"] = rng.bit_generator.random_raw(2)
    np.savez_compressed(HERE / "datagen.npz", **out)
    print("wrote", HERE / "datagen.npz", {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
