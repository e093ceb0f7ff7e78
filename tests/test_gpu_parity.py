"""Parity of the B200 path (through the C ABI) with the CPU oracle and with the
golden vectors of the reference.  Bar: bit-exact norms / probabilities /
score sums / budgets / sampled indices / scales; C.D within 1e-12 relative
(float64).  Marked gpu: runs on the B200 box only."""
import numpy as np
import pytest

import workloads
from golden_cases import make_instance, ssm_draws
from oracle import blockmm_oracle as O

pytestmark = pytest.mark.gpu

bm = pytest.importorskip("paper_2105_04940_b200")


def rel(a, b):
    d = np.linalg.norm(np.asarray(a) - np.asarray(b))
    r = np.linalg.norm(np.asarray(b))
    return d / r if r else d


# ---------------------------------------------------------------- norms


@pytest.mark.parametrize("m,n,p", [(1, 1, 1), (3, 7, 5), (200, 10000, 200), (17, 333, 129), (64, 1000, 1000),
                                   (5, 40, 16384), (2, 9, 257), (33, 130, 127)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_norms_bit_exact(m, n, p, dtype):
    g = np.random.default_rng(m * 1000 + n + p)
    M = (g.standard_normal((m, n)) * g.lognormal(0, 2, n)).astype(dtype)
    N = (g.standard_normal((n, p)) * g.lognormal(0, 2, (n, 1))).astype(dtype)
    cn = bm.column_norms(M)
    rn = bm.row_norms(N)
    assert np.array_equal(cn, np.sqrt(O.colsq(M.astype(np.float64))))
    assert np.array_equal(rn, np.sqrt(O.rowsq(N.astype(np.float64))))


@pytest.mark.parametrize("p,dtype", [(8, np.float32), (100, np.float64), (128, np.float32), (130, np.float64),
                                     (256, np.float32), (500, np.float64), (1000, np.float64), (4096, np.float32),
                                     (16384, np.float32), (6000, np.float64), (33, np.float64), (1001, np.float32),
                                     (4097, np.float64), (12345, np.float64), (16383, np.float32)])
def test_rowsq_staged_bit_exact(p, dtype):
    """The bulk-copy staged row kernel (inputs >= 8 MB, contiguous 16-byte rows),
    batched with a problem stride, against NumPy's pairwise order."""
    import torch
    g = np.random.default_rng(p)
    itemsize = np.dtype(dtype).itemsize
    n = max(64, (12 << 20) // (p * itemsize * 2))
    N = (g.standard_normal((2, n, p)) * g.lognormal(0, 2, (2, n, 1))).astype(dtype)
    Nd = torch.as_tensor(N, device="cuda")
    rs = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    from paper_2105_04940_b200 import _lib
    _lib.call("bmm_norms", _lib.matrix_dtype(Nd), None, 0, n, 0, 0, Nd.data_ptr(), p, p, n * p, 2, 0, None,
              rs.data_ptr(), _lib.stream_ptr())
    ref = np.concatenate([O.rowsq(N[b].astype(np.float64)) for b in range(2)])
    assert np.array_equal(rs.cpu().numpy(), ref)


@pytest.mark.parametrize("p,ld,dtype", [(500, 504, np.float64), (1000, 1024, np.float32), (300, 302, np.float64)])
def test_rowsq_padded_rows_bit_exact(p, ld, dtype):
    """Rows with a leading dimension larger than p (padded, 16-byte pitch or not)."""
    import torch
    g = np.random.default_rng(p + ld)
    itemsize = np.dtype(dtype).itemsize
    n = (20 << 20) // (ld * itemsize * 2)
    full = g.standard_normal((2, n, ld)).astype(dtype)
    Nd = torch.as_tensor(full, device="cuda")
    rs = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    from paper_2105_04940_b200 import _lib
    _lib.call("bmm_norms", _lib.matrix_dtype(Nd), None, 0, n, 0, 0, Nd.data_ptr(), p, ld, n * ld, 2, 0, None,
              rs.data_ptr(), _lib.stream_ptr())
    ref = np.concatenate([O.rowsq(full[b, :, :p].astype(np.float64)) for b in range(2)])
    assert np.array_equal(rs.cpu().numpy(), ref)


def test_norms_unaligned_view():
    import torch
    g = np.random.default_rng(4)
    M = g.standard_normal((11, 37))
    t = torch.as_tensor(M, device="cuda")[:, 1:]  # odd column offset -> scalar path
    cn = bm.column_norms(t).cpu().numpy()
    assert np.array_equal(cn, np.sqrt(O.colsq(M[:, 1:])))


# ---------------------------------------------------------------- golden small cases


def test_small_cases_against_reference_golden(golden_meta, golden_small):
    for case in golden_meta["cases"]:
        M, N = make_instance(case)
        g = {k.split("__", 1)[1]: v for k, v in golden_small.items() if k.startswith(case["name"] + "__")}
        part = bm.BlockPartition(tuple(case["sizes"]))
        c, c0, seed = case["c"], case["c0"], case["sample_seed"]
        name = case["name"]
        assert np.array_equal(bm.column_norms(M), g["colnorm"]), name
        assert np.array_equal(bm.row_norms(N), g["rownorm"]), name
        assert np.array_equal(bm.score_sums(M, N, part), g["s"]), name
        assert np.array_equal(np.concatenate(bm.optimal_probabilities(M, N, part).per_block), g["probs"]), name
        for meth, fn in (("OPL", bm.allocate_optimal), ("ONC", bm.allocate_by_score_sums)):
            plan = fn(M, N, part, c)
            assert np.array_equal(plan.budgets, g[f"{meth}_budgets"]), (name, meth)
            pair, prod, log = bm.estimate_product(M, N, plan, np.random.default_rng(seed))
            assert np.array_equal(log.column, g[f"{meth}_columns"]), (name, meth)
            assert np.array_equal(log.scale, g[f"{meth}_scale"]), (name, meth)
            assert rel(prod, g[f"{meth}_CD"]) < 1e-12, (name, meth)
        plan = bm.allocate_uniform(part, c)
        assert np.array_equal(plan.budgets, g["UU_budgets"])
        _, prod, log = bm.estimate_product(M, N, plan, np.random.default_rng(seed))
        assert np.array_equal(log.column, g["UU_columns"])
        assert rel(prod, g["UU_CD"]) < 1e-12
        for meth, pilot in (("ONU", "uniform"), ("ONMCNR", "norm")):
            res = bm.estimate_product_two_step(M, N, part, c, c0, np.random.default_rng(seed), pilot=pilot)
            assert res.plan.method == meth
            assert np.array_equal(res.plan.budgets, g[f"{meth}_budgets"]), (name, meth)
            np.testing.assert_allclose(res.plan.pilot_norms, g[f"{meth}_pilot"], rtol=1e-12, atol=0)
            assert np.array_equal(res.log.column, g[f"{meth}_columns"]), (name, meth)
            assert rel(res.product, g[f"{meth}_CD"]) < 1e-12
        draws = ssm_draws(case)
        np.testing.assert_allclose(bm.block_norm_probabilities(M, N, part), g["SSM_q"], rtol=1e-13)
        pair, prod, rec = bm.estimate_product_block_sampling(M, N, part, draws, np.random.default_rng(seed))
        assert np.array_equal(rec.blocks, g["SSM_blocks"]), name
        np.testing.assert_allclose(rec.scales, g["SSM_scale"], rtol=1e-13)
        assert rel(prod, g["SSM_CD"]) < 1e-12


def test_integerize_known_answers(golden_meta):
    for case in golden_meta["integerize"]:
        w = np.array(case["w"])
        caps = None if case["caps"] is None else np.array(case["caps"])
        floors = None if case["floors"] is None else np.array(case["floors"])
        if case["err"] == "ValueError":
            with pytest.raises(ValueError):
                bm.integerize(w, case["c"], caps=caps, floor=floors)
        elif case["err"] == "AssertionError":
            with pytest.raises(AssertionError):
                bm.integerize(w, case["c"], caps=caps, floor=floors)
        else:
            assert bm.integerize(w, case["c"], caps=caps, floor=floors).tolist() == case["out"], case


def test_integerize_large_random_vs_oracle():
    g = np.random.default_rng(8)
    for K in (1, 7, 64, 300, 1000, 4096):
        for _ in range(3):
            w = g.lognormal(0, 2, K) * (g.random(K) > 0.1)
            if w.sum() == 0:
                w[0] = 1.0
            caps = g.integers(1, 40, K)
            floors = w > 0
            lo, hi = int(floors.sum()), int(np.minimum(caps, 10**9).sum())
            c = int(g.integers(lo, hi + 1))
            assert np.array_equal(bm.integerize(w, c, caps=caps), O.integerize(w, c, caps, None))
            c2 = int(g.integers(K, 50 * K))
            assert np.array_equal(bm.integerize(w, c2, floor=np.zeros(K, bool)),
                                  O.integerize(w, c2, None, np.zeros(K, bool)))


# ---------------------------------------------------------------- full-size configs


def test_cfg1_against_golden(golden_cfg1):
    M, N, sizes = workloads.cfg1()
    part = bm.BlockPartition(sizes)
    g = golden_cfg1
    assert np.array_equal(np.concatenate(bm.optimal_probabilities(M, N, part).per_block), g["probs"])
    for meth, fn in (("OPL", bm.allocate_optimal), ("ONC", bm.allocate_by_score_sums)):
        plan = fn(M, N, part, 2000)
        assert np.array_equal(plan.budgets, g[f"{meth}_budgets"])
        _, prod, log = bm.estimate_product(M, N, plan, workloads.sample_rng(1))
        assert np.array_equal(log.column, g[f"{meth}_columns"])
        assert np.array_equal(log.scale, g[f"{meth}_scale"])
        assert rel(prod, g[f"{meth}_CD"]) < 1e-12
    _, prod, rec = bm.estimate_product_block_sampling(M, N, part, 20, workloads.sample_rng(1))
    assert np.array_equal(rec.blocks, g["SSM_blocks"])
    assert rel(prod, g["SSM_CD"]) < 1e-12


def test_cfg2_against_golden(golden_cfg2):
    M, N, sizes = workloads.cfg2()
    part = bm.BlockPartition(sizes)
    g = golden_cfg2
    for c_blocks, W in zip((10, 20, 40), (4000, 8000, 16000)):
        for meth in ("OPL", "ONC", "ONMCNR"):
            rng = workloads.sample_rng(2, c_blocks)
            if meth == "ONMCNR":
                res = bm.estimate_product_two_step(M, N, part, W, 500, rng, pilot="norm")
                plan, prod, log = res.plan, res.product, res.log
                np.testing.assert_allclose(plan.pilot_norms, g[f"{meth}_{W}_pilot"], rtol=1e-11)
            else:
                fn = bm.allocate_optimal if meth == "OPL" else bm.allocate_by_score_sums
                plan = fn(M, N, part, W)
                _, prod, log = bm.estimate_product(M, N, plan, rng)
            assert np.array_equal(plan.budgets, g[f"{meth}_{W}_budgets"]), (meth, W)
            assert np.array_equal(log.column, g[f"{meth}_{W}_columns"]), (meth, W)
            assert np.array_equal(log.scale, g[f"{meth}_{W}_scale"]), (meth, W)
            assert rel(prod[::7, ::7], g[f"{meth}_{W}_CDsub"]) < 1e-12
            assert abs(np.linalg.norm(prod) / g[f"{meth}_{W}_CDfrob"] - 1) < 1e-12


@pytest.mark.slow
def test_cfg3_two_step_against_oracle():
    M, N, sizes = workloads.cfg3()
    part = bm.BlockPartition(sizes)
    res = bm.estimate_product_two_step(M, N, part, 20000, 5000, workloads.sample_rng(3), pilot="uniform")
    ref = O.approx_product(M, N, sizes, 20000, "ONU", workloads.sample_rng(3), c0=5000)
    np.testing.assert_allclose(res.plan.pilot_norms, np.sqrt(ref["pilot_sq"]), rtol=1e-11)
    assert np.array_equal(res.plan.budgets, ref["budgets"])
    assert np.array_equal(res.log.column, ref["columns"])
    assert np.array_equal(res.log.scale, ref["scale"])
    assert rel(res.product, ref["CD"]) < 1e-12


# ---------------------------------------------------------------- reference edge cases


def test_sketch_bitwise_gather_and_record():
    g = np.random.default_rng(2)
    Mb = g.standard_normal((4, 6))
    Nb = g.standard_normal((6, 3))
    sc = np.sqrt(O.colsq(Mb)) * np.sqrt(O.rowsq(Nb))
    probs = sc / sc.sum()
    rng_a, rng_b = np.random.default_rng(5), np.random.default_rng(5)
    C, D, rec = bm.sketch_columns(Mb, Nb, 9, probs, rng_a)
    idx = O.draw(probs, 9, rng_b)
    assert np.array_equal(rec.columns, idx)
    for t in range(9):
        i = rec.columns[t]
        assert rec.probs[t] == probs[i]
        assert rec.scales[t] == 1.0 / np.sqrt(9 * probs[i])
        assert np.array_equal(C[:, t], Mb[:, i] * rec.scales[t])
        assert np.array_equal(D[t, :], Nb[i, :] * rec.scales[t])
    assert rng_a.bit_generator.state == rng_b.bit_generator.state  # caller stream advanced identically


def test_sketch_one_hot_and_zero_probability_columns():
    g = np.random.default_rng(0)
    Mb = g.standard_normal((3, 4))
    Nb = g.standard_normal((4, 2))
    C, D, rec = bm.sketch_columns(Mb, Nb, 8, np.array([0.0, 1.0, 0.0, 0.0]), np.random.default_rng(8))
    assert (rec.columns == 1).all()
    np.testing.assert_allclose(C @ D, np.outer(Mb[:, 1], Nb[1, :]), atol=1e-12)
    _, _, rec = bm.sketch_columns(Mb, Nb, 200, np.array([0.5, 0.0, 0.25, 0.25]), np.random.default_rng(3))
    assert set(np.unique(rec.columns)) <= {0, 2, 3}


def test_sketch_validation():
    g = np.random.default_rng(4)
    Mb, Nb = g.standard_normal((2, 3)), g.standard_normal((3, 2))
    ok = np.full(3, 1 / 3)
    rng = np.random.default_rng(1)
    for args in [(Mb, Nb, 0, ok), (Mb, Nb, 2, np.full(4, 0.25)), (Mb, Nb, 2, np.array([0.5, 0.3, 0.1])),
                 (Mb, Nb, 2, np.array([0.5, 0.7, -0.2])), (Mb, Nb[:2], 2, ok), (Mb, Nb, 2, np.zeros(3))]:
        with pytest.raises(ValueError):
            bm.sketch_columns(*args, rng)


def test_single_column_blocks_exact_product():
    g = np.random.default_rng(12)
    M, N = g.standard_normal((3, 5)), g.standard_normal((5, 4))
    part = bm.BlockPartition((1, 1, 1, 1, 1))
    plan = bm.allocate_uniform(part, 5)
    _, prod, log = bm.estimate_product(M, N, plan, np.random.default_rng(6))
    assert (log.scale == 1.0).all()
    # C is M and D is N exactly, so the product equals the device exact product bit for bit
    assert np.array_equal(prod, bm.multiply_exact(M, N))


def test_zero_block_skipped_and_caps():
    g = np.random.default_rng(16)
    M, N = g.standard_normal((2, 6)), g.standard_normal((6, 2))
    M[:, 2:4] = 0.0
    part = bm.BlockPartition.equal(6, 3)
    plan = bm.allocate_optimal(M, N, part, c=4)
    assert plan.budgets[1] == 0
    _, product, log = bm.estimate_product(M, N, plan, np.random.default_rng(8))
    assert set(np.unique(log.block)) <= {0, 2} and len(log) == plan.total
    with pytest.raises(ValueError):
        bm.allocate_optimal(M, N, part, c=5)
    nocap = bm.allocate_optimal(M, N, part, c=5, cap=False)
    assert nocap.budgets[1] == 0 and nocap.total == 5


def test_allocator_fallback_and_errors():
    M = np.array([[1.0, 0.0], [0.0, 2.0]])
    N = np.array([[3.0, 0.0], [0.0, 1.0]])
    plan = bm.allocate_optimal(M, N, bm.BlockPartition((1, 1)), 2, cap=False)
    assert plan.total == 2 and plan.notes
    plan = bm.allocate_by_score_sums(np.array([[3.0, 1.0]]), np.eye(2), bm.BlockPartition((1, 1)), 8, cap=False)
    assert list(plan.budgets) == [6, 2]
    with pytest.raises(ValueError):
        bm.allocate_by_score_sums(np.zeros((2, 4)), np.ones((4, 2)), bm.BlockPartition((2, 2)), 4)
    with pytest.raises(ValueError, match="required floors"):
        M, N, sizes = workloads.cfg1()
        bm.allocate_optimal(M, N, bm.BlockPartition(sizes), 20)
    assert list(bm.allocate_uniform(bm.BlockPartition((4, 4, 4)), 10).budgets) == [4, 3, 3]
    assert list(bm.integerize(np.ones(3), 10)) == [4, 3, 3]
    assert list(bm.integerize(np.array([0.7, 0.3]), 10, caps=np.array([5, 100]))) == [5, 5]
    assert list(bm.integerize(np.array([5.0, 0.0]), 6, floor=np.array([True, True]))) == [5, 1]


def test_two_step_validation_and_single_block():
    g = np.random.default_rng(18)
    M, N = g.standard_normal((3, 8)), g.standard_normal((8, 3))
    part = bm.BlockPartition.equal(8, 2)
    with pytest.raises(ValueError):
        bm.estimate_product_two_step(M, N, part, 6, 4, np.random.default_rng(1), pilot="x")
    with pytest.raises(ValueError):
        bm.estimate_product_two_step(M, N, part, 6, 1, np.random.default_rng(1))
    res = bm.estimate_product_two_step(M[:, :4], N[:4], bm.BlockPartition((4,)), 3, 2, np.random.default_rng(22))
    assert tuple(res.plan.budgets) == (3,)


def test_block_sampling_validation_and_degenerate():
    g = np.random.default_rng(27)
    M, N = g.standard_normal((2, 4)), g.standard_normal((4, 2))
    part = bm.BlockPartition.equal(4, 2)
    pair, product, rec = bm.estimate_product_block_sampling(M, N, part, 3, np.random.default_rng(28),
                                                            probs=np.array([1.0, 0.0]))
    assert (rec.blocks == 0).all() and pair.offsets[-1] == 6
    np.testing.assert_allclose(product, M[:, :2] @ N[:2], atol=1e-12)
    with pytest.raises(ValueError):
        bm.estimate_product_block_sampling(M, N, part, 0, np.random.default_rng(31))
    with pytest.raises(ValueError):
        bm.estimate_product_block_sampling(M, N, part, 2, np.random.default_rng(31), probs=np.array([0.7, 0.4]))
    with pytest.raises(ValueError):
        bm.block_norm_probabilities(np.zeros((2, 4)), np.zeros((4, 2)), part)


def test_determinism_and_spawn_side_effect():
    g = np.random.default_rng(15)
    M, N = g.standard_normal((3, 8)), g.standard_normal((8, 2))
    part = bm.BlockPartition.equal(8, 4)
    plan = bm.allocate_optimal(M, N, part, c=8)
    r1, r2 = np.random.default_rng(99), np.random.default_rng(99)
    p1 = bm.estimate_product(M, N, plan, r1)
    p2 = bm.estimate_product(M, N, plan, r2)
    assert np.array_equal(p1[1], p2[1]) and np.array_equal(p1[0].C, p2[0].C)
    # a second call on the same generator uses the next children, like the reference
    q1 = bm.estimate_product(M, N, plan, r1)
    ref_rng = np.random.default_rng(99)
    O_first = O.approx_product(M, N, part.sizes, 8, "OPL", ref_rng)
    O_second = O.approx_product(M, N, part.sizes, 8, "OPL", ref_rng)
    assert np.array_equal(p1[2].column, O_first["columns"])
    assert np.array_equal(q1[2].column, O_second["columns"])


# ---------------------------------------------------------------- GEMM / error kernels


@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (3, 5, 7), (64, 16, 64), (65, 17, 63), (200, 2000, 200),
                                   (500, 4001, 500), (8, 100000, 8), (130, 3, 257)])
def test_exact_product(m, k, n):
    g = np.random.default_rng(m + k + n)
    A, B = g.standard_normal((m, k)), g.standard_normal((k, n))
    out = bm.multiply_exact(A, B)
    assert rel(out, A @ B) < 1e-13


def test_block_scores_and_relative_error():
    g = np.random.default_rng(5)
    M, N = g.standard_normal((70, 333)), g.standard_normal((333, 90))
    sizes = (17, 100, 1, 215)
    sc = bm.block_scores(M, N, bm.BlockPartition(sizes))
    np.testing.assert_allclose(sc.product_norms ** 2, O.block_product_sq(M, N, sizes), rtol=1e-12)
    A = M @ N
    Bm = A + 1e-3 * g.standard_normal(A.shape)
    e, r = O.frob_errors(A, Bm)
    assert abs(bm.relative_error(Bm, A) - np.sqrt(e) / np.sqrt(r)) < 1e-14


@pytest.mark.parametrize("m,k,n,batch,shared_ref", [(200, 2000, 200, 7, True), (40, 64, 40, 33, False),
                                                    (65, 17, 63, 3, True), (130, 30000, 257, 1, False),
                                                    (500, 4001, 500, 2, True)])
def test_fused_error_epilogue(m, k, n, batch, shared_ref):
    """K9 (bmm_gemm_f64_err): ||ref - A B||_F^2 from the contraction's epilogue (single-pass
    tiles and split-K), with and without writing the product -- against NumPy (1e-12) and the
    plain contraction (the written product is bit-identical, the error sums equal)."""
    import torch
    from paper_2105_04940_b200 import _lib
    g = np.random.default_rng(m + k + n + batch)
    A, B = g.standard_normal((batch, m, k)), g.standard_normal((batch, k, n))
    exact = A @ B
    ref = (exact[0] if shared_ref else exact) + 1e-3 * g.standard_normal((m, n) if shared_ref else (batch, m, n))
    want = np.array([np.sum(((ref if shared_ref else ref[b]) - exact[b]) ** 2) for b in range(batch)])
    Ad, Bd, Rd = _lib.f64(A), _lib.f64(B), _lib.f64(ref)
    lib = _lib.load()
    ws = _lib.workspace(max(lib.bmm_gemm_f64_err_workspace(m, n, k, batch), lib.bmm_gemm_f64_workspace(m, n, k, batch)))
    plain = torch.empty((batch, m, n), dtype=torch.float64, device="cuda")
    _lib.call("bmm_gemm_f64", _lib.ptr(Ad), k, m * k, _lib.ptr(Bd), n, k * n, m, n, k, batch, _lib.ptr(plain), n, m * n,
              _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    errs = []
    for write in (True, False):
        out = torch.full((batch, m, n), -7.0, dtype=torch.float64, device="cuda")
        err = torch.empty(batch, dtype=torch.float64, device="cuda")
        _lib.call("bmm_gemm_f64_err", _lib.ptr(Ad), k, m * k, _lib.ptr(Bd), n, k * n, m, n, k, batch, _lib.ptr(Rd), n,
                  0 if shared_ref else m * n, _lib.ptr(out) if write else None, n, m * n, _lib.ptr(err), _lib.ptr(ws),
                  ws.numel(), _lib.stream_ptr())
        if write:
            assert torch.equal(out, plain)
        else:
            assert bool((out == -7.0).all())  # the product is never stored
        errs.append(err.cpu().numpy())
        np.testing.assert_allclose(errs[-1], want, rtol=1e-9)
    assert np.array_equal(errs[0], errs[1])


def test_fused_gather_kernels_match_materialised_sketch():
    """bmm_gemm_f64_gather / bmm_segsq_f64_gather == gather + GEMM / segsq (float64 rounding level)."""
    import torch
    from paper_2105_04940_b200 import _lib
    g = np.random.default_rng(31)
    m, n, p, W = 70, 900, 50, 333
    M = torch.as_tensor(g.standard_normal((m, n)), device="cuda")
    N = torch.as_tensor(g.standard_normal((n, p)), device="cuda")
    col = torch.as_tensor(g.integers(0, n, W), device="cuda")
    sc = torch.as_tensor(g.random(W) + 0.5, device="cuda")
    st = _lib.stream_ptr()
    C = torch.empty((m, W), dtype=torch.float64, device="cuda")
    D = torch.empty((W, p), dtype=torch.float64, device="cuda")
    _lib.call("bmm_gather", 0, 0, M.data_ptr(), n, 0, N.data_ptr(), p, 0, m, p, col.data_ptr(), sc.data_ptr(), W, W,
              1, C.data_ptr(), W, 0, D.data_ptr(), p, 0, st)
    ws = _lib.workspace(1 << 26)
    ref = torch.empty((m, p), dtype=torch.float64, device="cuda")
    out = torch.empty_like(ref)
    _lib.call("bmm_gemm_f64", C.data_ptr(), W, 0, D.data_ptr(), p, 0, m, p, W, 1, ref.data_ptr(), p, 0,
              ws.data_ptr(), ws.numel(), st)
    _lib.call("bmm_gemm_f64_gather", M.data_ptr(), n, 0, N.data_ptr(), p, 0, m, p, col.data_ptr(), sc.data_ptr(),
              W, W, 1, out.data_ptr(), p, 0, ws.data_ptr(), ws.numel(), st)
    assert ((out - ref).norm() / ref.norm()).item() < 1e-14
    seg = torch.as_tensor(np.array([0, 7, 7, 100, 333]), device="cuda")
    g_ref = torch.empty(4, dtype=torch.float64, device="cuda")
    g_out = torch.empty_like(g_ref)
    _lib.call("bmm_segsq_f64", C.data_ptr(), W, 0, D.data_ptr(), p, 0, m, p, seg.data_ptr(), 4, 0, 1,
              g_ref.data_ptr(), ws.data_ptr(), ws.numel(), st)
    _lib.call("bmm_segsq_f64_gather", M.data_ptr(), n, 0, N.data_ptr(), p, 0, m, p, col.data_ptr(), sc.data_ptr(),
              W, seg.data_ptr(), 4, 0, 1, g_out.data_ptr(), ws.data_ptr(), ws.numel(), st)
    np.testing.assert_allclose(g_out.cpu().numpy(), g_ref.cpu().numpy(), rtol=1e-13)
    assert g_ref[1].item() == 0.0


# ---------------------------------------------------------------- OPL weights

@pytest.mark.parametrize("case", ["cfg1", "unequal", "rank1"])
def test_optimal_size_weights_and_real_budgets(case):
    """optimal_size_weights = sqrt(max(s^2 - g^2, 0)) and real_optimal_budgets =
    c w / sum(w) (reference plan.py:350-370) against the oracle's s (exact order)
    and g (BLAS order: tolerance-level, 1e-12); the rank-1 case has g_k = s_k in
    exact arithmetic (radicand at the rounding slack, clamped to ~0)."""
    g = np.random.default_rng(77)
    if case == "cfg1":
        M, N = g.standard_normal((60, 1000)), g.standard_normal((1000, 50))
        sizes = (100,) * 10
    elif case == "unequal":
        M = g.standard_normal((40, 700)) * g.lognormal(0, 1.5, 700)
        N = g.standard_normal((700, 30)) * g.lognormal(0, 1.5, (700, 1))
        sizes = (1, 99, 300, 50, 250)
    else:  # every block's product M^k N_k is a sum of rank-1 terms u v^T: g_k = s_k
        u, v = g.standard_normal(20), g.standard_normal(30)
        a, b = g.lognormal(0, 1, 200), g.lognormal(0, 1, 200)
        M, N = np.outer(u, a), np.outer(b, v)
        sizes = (50,) * 4
    part = bm.BlockPartition(sizes)
    cs, rs = O.colsq(M), O.rowsq(N)
    _, s = O.block_stats(cs, rs, sizes)
    gsq = O.block_product_sq(M, N, sizes)
    w_ref = np.sqrt(np.maximum(s ** 2 - gsq, 0.0))
    w = bm.optimal_size_weights(M, N, part)
    if case == "rank1":
        assert np.all(w <= 1e-6 * s) and np.all(w_ref <= 1e-6 * s)
        return
    assert rel(w, w_ref) < 1e-12
    r = bm.real_optimal_budgets(M, N, part, 40)
    assert abs(r.sum() - 40) < 1e-9 and rel(r, 40 * w_ref / w_ref.sum()) < 1e-12


def test_staged_host_transfers_round_trip(monkeypatch):
    """Large numpy <-> device transfers of the drop-in API go through two pinned staging
    buffers with a threaded memcpy (_lib._upload / _lib.host): exact round trips for sizes
    that are not multiples of the chunk, every dtype the API moves."""
    import torch
    from paper_2105_04940_b200 import _lib
    monkeypatch.setattr(_lib, "_BIG", 1 << 20)
    monkeypatch.setattr(_lib, "_CHUNK", 300_000)
    g = np.random.default_rng(9)
    for shape, dt in (((1031, 517), np.float64), ((777, 1213), np.float32), ((400_003,), np.int64)):
        a = (g.standard_normal(shape) * 1000).astype(dt)
        d = _lib.to_device(a)
        assert d.is_cuda and tuple(d.shape) == shape and np.array_equal(d.cpu().numpy(), a)
        back = _lib.host(d)
        assert back.dtype == a.dtype and back.shape == a.shape and np.array_equal(back, a)
    small = g.standard_normal((10, 10))
    assert np.array_equal(_lib.host(_lib.to_device(small)), small)
    pinned = torch.from_numpy(g.standard_normal((600, 600))).pin_memory()
    assert torch.equal(_lib.to_device(pinned.numpy()).cpu(), pinned)
