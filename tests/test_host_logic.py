"""Host-side logic of the product package that runs without a GPU: generator
side effects, argument validation and record types."""
import numpy as np
import pytest

from oracle import numpy_rng as R
from paper_2105_04940_b200 import rng as hrng
from paper_2105_04940_b200.matrix import BlockPartition
from paper_2105_04940_b200.plan import BlockProbabilities, SamplingPlan, raise_status
from paper_2105_04940_b200 import _lib


@pytest.mark.parametrize("seed", [5, 2**70 + 3, [1, 2, 3]])
def test_spawn_words_match_numpy_children(seed):
    rng = np.random.default_rng(seed)
    rng.spawn(2)
    ref = np.random.default_rng(seed)
    ref.spawn(2)
    kids = ref.spawn(5)
    words, first = hrng.spawn_words(rng, 5)
    assert first == 2
    for j, kid in enumerate(kids):
        assert R.pool_from_assembled(list(map(int, words)) + [first + j]) == list(kid.bit_generator.seed_seq.pool)
    # side effect: the parent's counter advanced exactly like rng.spawn(5)
    assert rng.bit_generator.seed_seq.n_children_spawned == 7
    assert rng.spawn(1)[0].random() == ref.spawn(1)[0].random()


def test_spawn_words_nested_key():
    rng = np.random.default_rng(11)
    child = rng.spawn(2)[1]  # key (1,)
    words, first = hrng.spawn_words(child, 3)
    kid = np.random.default_rng(11).spawn(2)[1].spawn(3)[2]
    assert R.pool_from_assembled(list(map(int, words)) + [first + 2]) == list(kid.bit_generator.seed_seq.pool)


def test_consume_matches_random():
    a = np.random.default_rng(3)
    b = np.random.default_rng(3)
    a.integers(0, 2**32, dtype=np.uint32)  # leaves a buffered 32-bit half
    b.integers(0, 2**32, dtype=np.uint32)
    hrng.consume(a, 7)
    b.random(7)
    assert a.bit_generator.state == b.bit_generator.state
    st = hrng.stream_state(a)
    s = b.bit_generator.state["state"]
    assert (int(st[0]) << 64 | int(st[1])) == s["state"] and (int(st[2]) << 64 | int(st[3])) == s["inc"]


def test_non_pcg64_generator_rejected():
    with pytest.raises(ValueError):
        hrng.spawn_words(np.random.Generator(np.random.Philox(1)), 2)


def test_partition_and_plan_validation():
    part = BlockPartition((3, 5))
    assert part.offsets.tolist() == [0, 3, 8] and part.total == 8
    assert part.block_slice(1) == slice(3, 8)
    with pytest.raises(IndexError):
        part.block_slice(2)
    with pytest.raises(ValueError):
        BlockPartition(())
    with pytest.raises(ValueError):
        BlockPartition.equal(10, 3)
    probs = BlockProbabilities((np.full(3, 1 / 3), np.zeros(5)))
    assert probs.zero_blocks == (1,)
    SamplingPlan(part, probs, np.array([2, 0]))
    with pytest.raises(ValueError):
        SamplingPlan(part, probs, np.array([2, 1]))
    with pytest.raises(ValueError):
        BlockProbabilities((np.array([0.5, 0.4]),))


def test_status_mapping():
    raise_status(_lib.ST_OK, 0, 5)
    with pytest.raises(ValueError, match="below the 100 required floors"):
        raise_status(_lib.ST_BELOW_FLOORS, 100, 20)
    with pytest.raises(AssertionError):
        raise_status(_lib.ST_NOT_PLACED, 0, 1)
    with pytest.raises(ValueError, match="block 3: zero budget and zero-probability flag must coincide"):
        raise_status(_lib.ST_PLAN_MISMATCH, 3, 10)


def test_product_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2105_04940_b200 as bm
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        bm.column_norms(np.ones((2, 2)))


@pytest.mark.parametrize("method", ["ONC", "ONU"])
def test_seeds_from_keys_matches_generators(method):
    from paper_2105_04940_b200.pipeline import seeds_from_keys, seeds_from_rngs
    keys = np.array([0, 3, 4095])
    rngs = [np.random.default_rng(np.random.SeedSequence(210504940, spawn_key=(5, 1, int(k)))) for k in keys]
    a = seeds_from_rngs(method, rngs, 64)
    b = seeds_from_keys(method, 210504940, (5, 1), keys, 64)
    assert np.array_equal(a.main.words, b.main.words) and np.array_equal(a.main.first, b.main.first)
    if method == "ONU":
        assert np.array_equal(a.pilot.words, b.pilot.words) and np.array_equal(a.pilot.first, b.pilot.first)


# ---------------------------------------------------------------- matrix helpers

def test_as_matrix_coerces_and_validates():
    """as_matrix (reference matrix.py:21-32): float64, C-ordered, 2-D, finite."""
    from paper_2105_04940_b200.matrix import as_matrix
    a = as_matrix([[1, 2], [3, 4]])
    assert a.dtype == np.float64 and a.flags.c_contiguous and a.shape == (2, 2)
    f = np.asfortranarray(np.arange(6, dtype=np.float32).reshape(2, 3))
    b = as_matrix(f)
    assert b.flags.c_contiguous and b.dtype == np.float64 and np.array_equal(b, f)
    c = np.ones((3, 4))
    assert as_matrix(c) is c or np.shares_memory(as_matrix(c), c)  # already conforming: no copy
    with pytest.raises(ValueError, match="2-D"):
        as_matrix(np.ones(3))
    with pytest.raises(ValueError, match="2-D"):
        as_matrix(np.ones((2, 2, 2)))
    for bad in (np.nan, np.inf, -np.inf):
        x = np.ones((2, 2))
        x[1, 0] = bad
        with pytest.raises(ValueError, match="NaN or Inf"):
            as_matrix(x)


def test_block_partition_contract():
    """BlockPartition (reference matrix.py:35-79): sizes, equal(), offsets, block_slice."""
    p = BlockPartition((3, 1, 4))
    assert p.num_blocks == 3 and p.total == 8
    assert list(p.offsets) == [0, 3, 4, 8] and p.offsets.dtype == np.int64
    assert p.block_slice(2) == slice(4, 8)
    with pytest.raises(IndexError):
        p.block_slice(3)
    with pytest.raises(IndexError):
        p.block_slice(-1)
    assert BlockPartition.equal(12, 4).sizes == (3, 3, 3, 3)
    with pytest.raises(ValueError):
        BlockPartition.equal(10, 4)
    with pytest.raises(ValueError):
        BlockPartition(())
    with pytest.raises(ValueError):
        BlockPartition((2, 0, 1))
    with pytest.raises(ValueError, match="partition covers"):
        p.check_length(9)


def test_block_view_zero_copy():
    """block_view (reference matrix.py:82-95): views, never copies; axis and length checks."""
    from paper_2105_04940_b200.matrix import block_view
    part = BlockPartition((2, 3, 1))
    M = np.arange(4 * 6, dtype=np.float64).reshape(4, 6)
    N = np.arange(6 * 5, dtype=np.float64).reshape(6, 5)
    v = block_view(M, part, 1, "columns")
    assert v.shape == (4, 3) and np.shares_memory(v, M) and np.array_equal(v, M[:, 2:5])
    w = block_view(N, part, 2, "rows")
    assert w.shape == (1, 5) and np.shares_memory(w, N) and np.array_equal(w, N[5:6])
    v[0, 0] = -1.0  # a view: writes show through
    assert M[0, 2] == -1.0
    with pytest.raises(ValueError, match="axis"):
        block_view(M, part, 0, "diagonal")
    with pytest.raises(ValueError, match="partition covers"):
        block_view(N, part, 0, "columns")
    with pytest.raises(IndexError):
        block_view(M, part, 3)


@pytest.mark.parametrize("count", [1, 5, 50, 64, 4096])
def test_advance_spawn_counter_equals_public_spawn(count):
    """rng.spawn(K)'s only lasting effect on the caller's generator is the parent's child
    counter (estimators.py:141,207; plan.py:456): the shortcut leaves the SeedSequence in the
    state the public call leaves it in -- same counter, entropy, key and pool, same next
    children -- for the first spawn and for a later one."""
    from paper_2105_04940_b200.rng import advance_spawn_counter
    a = np.random.SeedSequence(210504940, spawn_key=(2, 1, 7))
    b = np.random.SeedSequence(210504940, spawn_key=(2, 1, 7))
    for _ in range(2):
        advance_spawn_counter(a, count)
        b.spawn(count)
        assert a.n_children_spawned == b.n_children_spawned
        assert a.entropy == b.entropy and a.spawn_key == b.spawn_key and a.pool_size == b.pool_size
        assert np.array_equal(a.pool, b.pool)
        ca, cb = a.spawn(2), b.spawn(2)
        for x, y in zip(ca, cb):
            assert x.spawn_key == y.spawn_key and np.array_equal(x.generate_state(4), y.generate_state(4))
    advance_spawn_counter(a, 0)
    assert a.n_children_spawned == b.n_children_spawned
