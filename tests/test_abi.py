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


def test_cpp_dropin_header_compiles(tmp_path):
    """include/epikv/epikv_gpu.hpp compiles against the reference headers."""
    ref = "/root/reference/proj/include"
    if not os.path.isdir(ref):
        pytest.skip("reference headers absent")
    src = tmp_path / "t.cpp"
    src.write_text('#include "epikv/epikv_gpu.hpp"\nint main() { return 0; }\n')
    json_inc = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{ROOT}/include", f"-I{ref}", f"-I{json_inc}",
                        "-I/usr/local/cuda/include", str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def test_device_episode_header_is_standalone_cxx17():
    """include/epikv/epikv_device.hpp (the C++ throughput API) compiles on its
    own as C++17 against epk.h and the CUDA runtime headers only."""
    import shutil
    import subprocess
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    src = '#include "epikv/epikv_device.hpp"\nint main() { return sizeof(epikv::gpu::DeviceEpisode) > 0 ? 0 : 1; }\n'
    r = subprocess.run([gxx, "-std=c++17", "-fsyntax-only", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                        "-I", "/usr/local/cuda/include", "-x", "c++", "-"], input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "warning" not in r.stderr, r.stderr
