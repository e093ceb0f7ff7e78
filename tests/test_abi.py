"""The C-ABI library loads without a GPU and exports every symbol the header declares."""
import ctypes
import re

from conftest import ROOT


def declared_symbols():
    text = (ROOT / "include" / "blockmm_b200.h").read_text()
    body = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bmm_\w+)\s*\(", body)))


def test_library_exports_header_symbols():
    from paper_2105_04940_b200 import _lib
    assert _lib.LIB_PATH.exists(), "build the library first (python -m paper_2105_04940_b200.build)"
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the python binding table covers the whole header
    assert set(syms) == set(_lib.SIGNATURES)


def test_library_version_and_error_slot():
    from paper_2105_04940_b200 import _lib
    lib = _lib.load()
    assert lib.bmm_version() == 1
    assert isinstance(lib.bmm_last_error(), bytes)
    assert lib.bmm_launch_count() >= 0


def test_host_argument_errors_without_gpu():
    """Shape validation happens before any device work, so it runs on CPU."""
    from paper_2105_04940_b200 import _lib
    lib = _lib.load()
    rc = lib.bmm_norms(0, None, -1, 5, 5, 0, None, 0, 0, 0, 1, 0, None, None, None)
    assert rc == -1
    assert b"bad shape" in lib.bmm_last_error()
    assert lib.bmm_budgets_workspace(4096) > 0
