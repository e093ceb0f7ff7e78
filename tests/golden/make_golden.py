"""Generate the golden vectors that pin oracle/ (and, through it, the device path).

Runs the REFERENCE package itself (``blockmm`` from /root/reference/pkg/src),
so it only works in the build container; the outputs are committed as small
.npz / .json fixtures and travel to the GPU box.  Re-run with

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Inputs are regenerated from seeds in the tests, so only seeds and outputs
are stored.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import blockmm as ref  # noqa: E402  (the reference, read-only)

import workloads  # noqa: E402


def small_cases():
    """Seeded small instances with the edge cases the reference tests exercise."""
    cases = []
    rng = np.random.default_rng(20260101)
    specs = [
        ("tiny", 3, 8, 4, (3, 5)),
        ("unequal", 12, 300, 10, (17, 1, 64, 129, 2, 87)),
        ("equal", 7, 256, 9, (32,) * 8),
        ("wide", 5, 1000, 3, (200, 300, 500)),
        ("single", 4, 130, 6, (130,)),
    ]
    for name, m, n, p, sizes in specs:
        seed = int(rng.integers(1, 2**31))
        cases.append(dict(name=name, m=m, n=n, p=p, sizes=list(sizes), seed=seed, zero=None))
    # zero column inside a block and a whole zero block (M side)
    cases.append(dict(name="zeros", m=6, n=40, p=5, sizes=[10, 10, 10, 10], seed=77, zero=[[3], [20, 30]]))
    return cases


def make_instance(case):
    g = np.random.default_rng(case["seed"])
    M = g.standard_normal((case["m"], case["n"])) * g.lognormal(0, 1.0, case["n"])
    N = g.standard_normal((case["n"], case["p"]))
    if case["zero"]:
        cols, blk = case["zero"]
        M[:, cols] = 0.0
        M[:, blk[0]:blk[1]] = 0.0
    return M, N


def run_case(M, N, sizes, c, c0, seed):
    part = ref.BlockPartition(tuple(sizes))
    out = {}
    out["colnorm"] = ref.column_norms(M)
    out["rownorm"] = ref.row_norms(N)
    out["s"] = ref.score_sums(M, N, part)
    out["probs"] = np.concatenate(ref.optimal_probabilities(M, N, part).per_block)
    for meth, fn in (("OPL", ref.allocate_optimal), ("ONC", ref.allocate_by_score_sums)):
        plan = fn(M, N, part, c)
        out[f"{meth}_budgets"] = plan.budgets
        pair, prod, log = ref.estimate_product(M, N, plan, np.random.default_rng(seed))
        out[f"{meth}_columns"] = log.column
        out[f"{meth}_scale"] = log.scale
        out[f"{meth}_CD"] = prod
    plan = ref.allocate_uniform(part, c)
    out["UU_budgets"] = plan.budgets
    _, prod, log = ref.estimate_product(M, N, plan, np.random.default_rng(seed))
    out["UU_columns"] = log.column
    out["UU_CD"] = prod
    for meth, pilot in (("ONU", "uniform"), ("ONMCNR", "norm")):
        res = ref.estimate_product_two_step(M, N, part, c, c0, np.random.default_rng(seed), pilot=pilot)
        out[f"{meth}_budgets"] = res.plan.budgets
        out[f"{meth}_pilot"] = res.plan.pilot_norms
        out[f"{meth}_columns"] = res.log.column
        out[f"{meth}_CD"] = res.product
    draws = max(1, c // max(1, int(np.mean(sizes))))
    pair, prod, rec = ref.estimate_product_block_sampling(M, N, part, draws, np.random.default_rng(seed))
    out["SSM_draws"] = np.array(draws)
    out["SSM_q"] = ref.block_norm_probabilities(M, N, part)
    out["SSM_blocks"] = rec.blocks
    out["SSM_scale"] = rec.scales
    out["SSM_CD"] = prod
    return out


def main():
    meta = {"cases": []}
    arrays = {}
    for case in small_cases():
        M, N = make_instance(case)
        K = len(case["sizes"])
        nz_blocks = K if not case["zero"] else K - 1
        c = max(nz_blocks, min(sum(case["sizes"]) // 3, 3 * K + 5))
        c0 = 2 * K
        case.update(c=c, c0=c0, sample_seed=case["seed"] + 1)
        res = run_case(M, N, case["sizes"], c, c0, case["sample_seed"])
        for k, v in res.items():
            arrays[f"{case['name']}__{k}"] = np.asarray(v)
        meta["cases"].append(case)
    np.savez_compressed(HERE / "small_cases.npz", **arrays)

    # cfg1 at full size (inputs regenerated from workloads.cfg1)
    M, N, sizes = workloads.cfg1()
    part = ref.BlockPartition(sizes)
    g1 = {}
    for meth, fn in (("OPL", ref.allocate_optimal), ("ONC", ref.allocate_by_score_sums)):
        plan = fn(M, N, part, 2000)
        _, prod, log = ref.estimate_product(M, N, plan, workloads.sample_rng(1))
        g1[f"{meth}_budgets"] = plan.budgets
        g1[f"{meth}_columns"] = log.column
        g1[f"{meth}_scale"] = log.scale
        g1[f"{meth}_CD"] = prod
    g1["probs"] = np.concatenate(ref.optimal_probabilities(M, N, part).per_block)
    g1["s"] = ref.score_sums(M, N, part)
    _, prod, rec = ref.estimate_product_block_sampling(M, N, part, 20, workloads.sample_rng(1))
    g1["SSM_blocks"] = rec.blocks
    g1["SSM_CD"] = prod
    np.savez_compressed(HERE / "cfg1.npz", **g1)

    # cfg2 at full size: budgets / indices per c and method, CD subsampled
    M, N, sizes = workloads.cfg2()
    part = ref.BlockPartition(sizes)
    g2 = {"sizes": np.array(sizes)}
    for c_blocks, W in zip((10, 20, 40), (4000, 8000, 16000)):
        for meth in ("OPL", "ONC", "ONMCNR"):
            rng = workloads.sample_rng(2, c_blocks)
            if meth == "ONMCNR":
                res = ref.estimate_product_two_step(M, N, part, W, 500, rng, pilot="norm")
                plan, prod, log = res.plan, res.product, res.log
                g2[f"{meth}_{W}_pilot"] = plan.pilot_norms
            else:
                fn = ref.allocate_optimal if meth == "OPL" else ref.allocate_by_score_sums
                plan = fn(M, N, part, W)
                _, prod, log = ref.estimate_product(M, N, plan, rng)
            g2[f"{meth}_{W}_budgets"] = plan.budgets
            g2[f"{meth}_{W}_columns"] = log.column
            g2[f"{meth}_{W}_scale"] = log.scale
            g2[f"{meth}_{W}_CDsub"] = prod[::7, ::7]
            g2[f"{meth}_{W}_CDfrob"] = np.array(np.linalg.norm(prod))
    np.savez_compressed(HERE / "cfg2.npz", **g2)

    # integerize known answers (value or error class)
    ig = []
    r = np.random.default_rng(99)
    for _ in range(400):
        K = int(r.integers(1, 12))
        w = r.random(K) * (r.random(K) > 0.15)
        if w.sum() == 0:
            w[0] = 0.5
        caps = r.integers(0, 15, K) if r.random() < 0.6 else None
        floors = (r.random(K) < 0.5) if r.random() < 0.3 else None
        c = int(r.integers(0, 60))
        try:
            outv = ref.integerize(w, c, caps=caps, floor=floors).tolist()
            err = None
        except ValueError:
            outv, err = None, "ValueError"
        except AssertionError:
            outv, err = None, "AssertionError"
        ig.append(dict(w=w.tolist(), c=c, caps=None if caps is None else caps.tolist(),
                       floors=None if floors is None else floors.tolist(), out=outv, err=err))
    meta["integerize"] = ig

    # numpy stream known answers (PCG64 via SeedSequence children)
    kat = []
    for ent, key in [(5, ()), (12345, (0,)), (2**100 + 7, (1, 2, 3, 4, 5)), (workloads.ROOT, (1, 0, 3)),
                     (2**32, (2**33, 1)), ([1, 2, 3], (4,))]:
        ss = np.random.SeedSequence(ent, spawn_key=key)
        bg = np.random.PCG64(ss)
        st = bg.state["state"]
        g = np.random.Generator(bg)
        kat.append(dict(entropy=ent if isinstance(ent, int) else list(ent), key=list(key),
                        state=str(st["state"]), inc=str(st["inc"]),
                        raw=[str(x) for x in np.random.Generator(np.random.PCG64(
                            np.random.SeedSequence(ent, spawn_key=key))).bit_generator.random_raw(8)],
                        u=g.random(8).tolist()))
    meta["rng_kat"] = kat
    (HERE / "golden.json").write_text(json.dumps(meta, indent=1))
    print("wrote", sorted(p.name for p in HERE.iterdir()))


if __name__ == "__main__":
    main()
