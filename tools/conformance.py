"""Reference conformance gate: run the reference package's own
API tests -- test_matrix.py, test_plan.py, test_estimators.py from
pkg/tests -- against THIS package, with the module name ``blockmm`` aliased to
``paper_2105_04940_b200`` (and blockmm.matrix / .plan / .estimators to its
modules).  Needs a GPU (the package has no CPU fallback).

The reference's tests are not part of this repository.  To run the gate on the
GPU box, stage them next to the repo first (a git-ignored directory that
travels with gpurun):
    mkdir -p conformance_stage && cp /root/reference/pkg/tests/{conftest,oracles,test_matrix,test_plan,test_estimators}.py conformance_stage/
    gpurun -- 'python tools/conformance.py conformance_stage > gpurun_out/conformance.log 2>&1'
and delete the staging directory afterwards.  The log lists every test with its
outcome (pytest -rA); deviations are named in profiles/*_conformance.md."""
import importlib
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def alias():
    pkg = importlib.import_module("paper_2105_04940_b200")
    sys.modules["blockmm"] = pkg
    for sub in ("matrix", "plan", "estimators", "analysis", "datagen", "io"):
        sys.modules[f"blockmm.{sub}"] = importlib.import_module(f"paper_2105_04940_b200.{sub}")


def main(argv):
    stage = Path(argv[1] if len(argv) > 1 else ROOT / "conformance_stage").resolve()
    files = [str(stage / f) for f in ("test_matrix.py", "test_plan.py", "test_estimators.py")]
    missing = [f for f in files if not Path(f).exists()]
    if missing:
        print(f"reference tests not staged: {missing}")
        return 2
    alias()
    sys.path.insert(0, str(stage))
    return pytest.main([*files, "-q", "-rA", "-p", "no:cacheprovider", "--rootdir", str(stage),
                        "-o", "addopts=", "--tb=short"])


if __name__ == "__main__":
    sys.exit(main(sys.argv))
