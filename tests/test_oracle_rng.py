"""Pin the numpy stream restatement (oracle/numpy_rng.py, which the device
RNG in csrc/rng.cuh mirrors) against live numpy and committed KAT vectors."""
import numpy as np
import pytest

from oracle import numpy_rng as R


def test_committed_kat(golden_meta):
    for kat in golden_meta["rng_kat"]:
        ent = kat["entropy"]
        key = tuple(kat["key"])
        g = R.PCG64(ent, key)
        assert g.state == int(kat["state"]) and g.inc == int(kat["inc"])
        raws = [g.next64() for _ in range(8)]
        assert raws == [int(x) for x in kat["raw"]]
        g2 = R.PCG64(ent, key)
        assert [g2.random() for _ in range(8)] == kat["u"]


@pytest.mark.parametrize("ent,key", [(0, ()), (1, (0,)), (2**64 - 1, (3, 1)), (210504940, (5, 1, 4095)),
                                      ([7, 2**40], (9,)), (123, (2**32 + 5,))])
def test_live_numpy(ent, key):
    ss = np.random.SeedSequence(ent, spawn_key=key)
    assert list(ss.pool) == R.seed_pool(ent, key)
    gen = np.random.Generator(np.random.PCG64(ss))
    mine = R.PCG64(ent, key)
    assert [mine.random() for _ in range(64)] == gen.random(64).tolist()


def test_spawn_equivalence():
    parent = np.random.default_rng(np.random.SeedSequence(99, spawn_key=(1, 2)))
    parent.spawn(3)  # advance the child counter like an earlier estimate call
    kids = parent.spawn(4)
    for j, kid in enumerate(kids):
        mine = R.child_stream(99, (1, 2), 3 + j)
        assert [mine.random() for _ in range(5)] == kid.random(5).tolist()
