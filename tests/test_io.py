"""Wire and on-disk formats against files written by the
reference's own writers (tests/golden/io/, tests/golden/make_io_golden.py):
byte-identical output, identical parsed values."""
from pathlib import Path

import numpy as np
import pytest

from random_cases import sweep_params

torch = pytest.importorskip("torch")
bm = pytest.importorskip("paper_2105_04940_b200")
from paper_2105_04940_b200 import io as bio  # noqa: E402

IO = Path(__file__).resolve().parent / "golden" / "io"


def _instance():
    M, N, sizes, c, c0 = sweep_params(11)
    return M, N, sizes, c


def test_matrix_binary_and_csv_byte_identical(tmp_path):
    M, N, _, _ = _instance()
    bio.save_matrix(tmp_path / "M.bin", M)
    assert (tmp_path / "M.bin").read_bytes() == (IO / "M.bin").read_bytes()
    bio.save_matrix_csv(tmp_path / "M.csv", M)
    assert (tmp_path / "M.csv").read_bytes() == (IO / "M.csv").read_bytes()
    assert np.array_equal(bio.load_matrix(IO / "M.bin"), M)
    assert np.array_equal(bio.load_matrix_csv(IO / "M.csv"), M)
    Mi, Ni, doc = bio.load_instance(IO / "inst")
    assert np.array_equal(Mi, M) and np.array_equal(Ni, N) and doc["case"] == "sweep11"
    bio.save_instance(tmp_path / "inst", M, N, {"case": "sweep11", "seed": 1011})
    for f in ("inst.json", "inst_left.bin", "inst_right.bin"):
        assert (tmp_path / f).read_bytes() == (IO / f).read_bytes()


def test_matrix_format_errors(tmp_path):
    (tmp_path / "short.bin").write_bytes(b"\x01\x00")
    with pytest.raises(ValueError, match="truncated header"):
        bio.load_matrix(tmp_path / "short.bin")
    raw = (IO / "M.bin").read_bytes()
    (tmp_path / "cut.bin").write_bytes(raw[:-8])
    with pytest.raises(ValueError, match="expected"):
        bio.load_matrix(tmp_path / "cut.bin")
    (tmp_path / "e.csv").write_text("")
    with pytest.raises(ValueError, match="empty CSV"):
        bio.load_matrix_csv(tmp_path / "e.csv")
    with pytest.raises(ValueError, match="NaN or Inf"):
        bio.save_matrix(tmp_path / "x.bin", np.array([[1.0, np.nan]]))


@pytest.mark.parametrize("name", ["OPL", "ONC", "UU"])
def test_plan_json_roundtrip_byte_identical(name):
    text = (IO / f"plan_{name}_probs.json").read_text()
    plan = bm.plan_from_json(text)  # explicit probabilities: no factors needed
    assert bm.plan_to_json(plan, include_probs=True) == text
    assert bm.plan_to_json(plan) == (IO / f"plan_{name}.json").read_text()


def test_plan_json_errors():
    doc = bm.plan_to_dict(bm.plan_from_json((IO / "plan_UU_probs.json").read_text()))
    bad = dict(doc, total=doc["total"] + 1)
    with pytest.raises(ValueError, match="recorded total"):
        bm.plan_from_dict(bad)
    opt = bm.plan_to_dict(bm.plan_from_json((IO / "plan_OPL_probs.json").read_text()))
    opt.pop("probs", None)
    with pytest.raises(ValueError, match="requires the factor matrices"):
        bm.plan_from_dict(opt)


def test_sample_log_csv_byte_identical(tmp_path):
    rows = [line.split(",") for line in (IO / "log_OPL.csv").read_text().splitlines()[1:]]
    log = bm.SampleLog(np.array([int(r[1]) for r in rows]), np.array([int(r[2]) for r in rows]),
                       np.array([int(r[3]) for r in rows]), np.array([float(r[4]) for r in rows]),
                       np.array([float(r[5]) for r in rows]))
    log.write_csv(tmp_path / "log.csv", rep=3)
    assert (tmp_path / "log.csv").read_bytes() == (IO / "log_OPL.csv").read_bytes()


@pytest.mark.gpu
def test_device_io_and_plan_regeneration(tmp_path):
    M, N, sizes, c = _instance()
    Md = bio.load_matrix(IO / "M.bin", device=True)
    assert Md.is_cuda and np.array_equal(Md.cpu().numpy(), M)
    bio.save_matrix(tmp_path / "Md.bin", Md)
    assert (tmp_path / "Md.bin").read_bytes() == (IO / "M.bin").read_bytes()
    Mi, Ni, _ = bio.load_instance(IO / "inst", device=True)
    # 'optimal' rule: probabilities regenerated on device, identical to the reference's
    plan = bm.plan_from_json((IO / "plan_OPL.json").read_text(), Mi, Ni)
    assert bm.plan_to_json(plan, include_probs=True) == (IO / "plan_OPL_probs.json").read_text()
    ours = bm.allocate_optimal(M, N, bm.BlockPartition(sizes), c)
    assert bm.plan_to_json(ours) == (IO / "plan_OPL.json").read_text()
    _, _, log = bm.estimate_product(M, N, ours, np.random.default_rng(5))
    log.write_csv(tmp_path / "log.csv", rep=3)
    assert (tmp_path / "log.csv").read_bytes() == (IO / "log_OPL.csv").read_bytes()
