import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built C-ABI library")
    config.addinivalue_line("markers", "slow: full-size configuration checks")


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def golden_small():
    return dict(np.load(GOLDEN / "small_cases.npz"))


@pytest.fixture(scope="session")
def golden_cfg1():
    return dict(np.load(GOLDEN / "cfg1.npz"))


@pytest.fixture(scope="session")
def golden_cfg2():
    return dict(np.load(GOLDEN / "cfg2.npz"))
