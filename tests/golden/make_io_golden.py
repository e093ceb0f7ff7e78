"""Files written by the REFERENCE's own writers: matrix
binary/CSV (matrix.py:121-159), instance sidecar (datagen.py:113-132), plan
JSON (plan.py:499-555) and SampleLog CSV (estimators.py:111-116), for a small
seeded instance.  Build-container only; outputs committed under tests/golden/io/.

    python tests/golden/make_io_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
OUT = HERE / "io"
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import blockmm as ref  # noqa: E402  (the reference, read-only)
from blockmm import datagen  # noqa: E402

from random_cases import sweep_params  # noqa: E402


def main():
    OUT.mkdir(exist_ok=True)
    M, N, sizes, c, c0 = sweep_params(11)
    part = ref.BlockPartition(sizes)
    ref.save_matrix(OUT / "M.bin", M)
    ref.save_matrix_csv(OUT / "M.csv", M)
    datagen.save_instance(OUT / "inst", M, N, {"case": "sweep11", "seed": 1011})
    plans = {"OPL": ref.allocate_optimal(M, N, part, c), "ONC": ref.allocate_by_score_sums(M, N, part, c),
             "UU": ref.allocate_uniform(part, c)}
    for name, plan in plans.items():
        (OUT / f"plan_{name}.json").write_text(ref.plan_to_json(plan))
        (OUT / f"plan_{name}_probs.json").write_text(ref.plan_to_json(plan, include_probs=True))
    _, _, log = ref.estimate_product(M, N, plans["OPL"], np.random.default_rng(5))
    log.write_csv(OUT / "log_OPL.csv", rep=3)


if __name__ == "__main__":
    main()
