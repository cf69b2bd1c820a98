"""CPU-side checks of the C-ABI boundary (no GPU needed, no compute calls)."""
import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HDR = ROOT / "include" / "at_b200.h"


def declared_symbols():
    txt = HDR.read_text()
    return sorted(set(re.findall(r"^AT_API\s+[\w\s\*]+?\b(\w+)\s*\(", txt, flags=re.M)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1805_08166_b200 import build
    return build.build()


def test_header_declares_the_six_calls():
    syms = declared_symbols()
    for name in ("space_create", "features_extract", "gbt_predict", "sa_explore", "select_topk", "gbt_fit_hist"):
        assert name in syms


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", str(libpath)], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_resolves_without_gpu(libpath):
    lib = ctypes.CDLL(str(libpath))
    for s in declared_symbols():
        assert getattr(lib, s) is not None
    lib.at_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.at_last_error(), bytes)


def test_host_validation_needs_no_gpu(libpath):
    """Argument validation happens on the host before any CUDA call."""
    from paper_1805_08166_b200 import at
    L = at.lib()
    h = ctypes.c_void_p()
    assert L.space_create(None, 1, ctypes.byref(h)) == -1
    w = at.workload(kind=7)
    assert L.space_create(ctypes.byref(w), 1, ctypes.byref(h)) == -1
    assert b"kind" in L.at_last_error()
    assert L.features_extract(None, None, 0, None, 0, None) == -1
    assert L.gbt_predict(None, None, 0, 0, None, None, None) == -1


def test_product_package_does_not_import_the_oracle():
    pkg = ROOT / "paper_1805_08166_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        txt = f.read_text()
        assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
        assert "oracle.h" not in txt, f
