"""The C ABI library builds for sm_100a, loads without a GPU, and exports
every symbol include/epk/epk.h declares; the C++ drop-in header compiles."""
import os
import subprocess

import pytest

from paper_2509_17396_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_and_exports_header_symbols():
    lib = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 24
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.epk_version() == 10000
    assert lib.epk_status_string(-2).decode() == "pinned entries exceed layer budget"


def test_library_is_sm100a_native():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2509_17396_b200 as epk
    with pytest.raises(RuntimeError):
        epk.Context(0)
