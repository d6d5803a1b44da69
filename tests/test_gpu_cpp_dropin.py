"""The C++ drop-in (include/epikv/epikv_gpu.hpp) against the reference
library call for call: tests/cpp/test_dropin.cpp, built against the
reference headers in place by tests/cpp/Makefile (travels to the GPU box)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "test_dropin")


def test_cpp_dropin_matches_reference(gpu):
    if not os.path.exists(BIN):
        pytest.skip("C++ drop-in driver not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout


C_BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "abi_c_step")


def test_plain_c_abi_step(gpu):
    """include/epk/epk.h from plain C (gcc, no C++ / torch): one bf16 block step."""
    assert os.path.exists(C_BIN), "tests/cpp/_build/abi_c_step not built (tests/cpp/Makefile)"
    r = subprocess.run([C_BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "abi_c_step ok" in r.stdout


B_BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "test_build")


@pytest.mark.parametrize("nccl", [False, True])
def test_cpp_multi_gpu_build_matches_reference(gpu, nccl):
    """epikv::gpu::build (one thread + epk_ctx per device entry, episodes
    round-robin, optional sharded k-means) writes the reference build's bytes;
    with EPK_FORCE_NCCL=1 the one-device k-means chain goes through NCCL
    (ncclCommInitAll + ncclBroadcast, libnccl.so.2 loaded at run time)."""
    if not os.path.exists(B_BIN):
        pytest.skip("C++ build driver not built (needs /root/reference at build time)")
    env = dict(os.environ, EPK_FORCE_NCCL="1") if nccl else None
    r = subprocess.run([B_BIN], capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout


F_BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "test_forward")


def test_cpp_device_forward_matches_reference(gpu):
    """epikv::gpu::forward (epk_toy_forward) bit-identical to the
    reference forward with the softmax rows on the host, within 1e-13 with them
    on the device; gpu::block_prefill / measure_sensitivity with device forwards
    equal the reference; the timing line compares the three block loops."""
    if not os.path.exists(F_BIN):
        pytest.skip("C++ forward driver not built (needs /root/reference at build time)")
    r = subprocess.run([F_BIN, "--timing"], capture_output=True, text=True, timeout=1800)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout


D_BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "test_device_episode")


def test_cpp_device_episode_matches_reference(gpu):
    """epikv::gpu::DeviceEpisode (include/epikv/epikv_device.hpp), the C++ host
    API of the throughput path: 8 blocks of append -> fused tensor-core step,
    each equal to the reference's evict_to_budget on the step's own scores
    (entries, positions, widened bf16 keys / values); then the cfg2 workload
    timed from C++ (append + step per block)."""
    if not os.path.exists(D_BIN):
        pytest.skip("C++ device-episode driver not built (needs /root/reference at build time)")
    r = subprocess.run([D_BIN, "--timing", "50"], capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout
