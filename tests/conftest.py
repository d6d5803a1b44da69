"""Test configuration.

-m "not gpu": oracle vs reference / golden fixtures, host logic, C-ABI
              symbol checks, multi-process (gloo) host logic.  No GPU needed.
-m gpu:       parity of the sm_100a kernels (through the C ABI) against the
              oracle on a real B200.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as O
    O.orc()
    return O


@pytest.fixture(scope="session")
def ref(orc):
    if not orc.ref_available():
        pytest.skip("reference tree and oracle/_ref absent (GPU box without /root/reference)")
    orc.ref()
    return orc


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    import paper_2509_17396_b200 as epk
    from paper_2509_17396_b200 import _lib
    _lib.load()
    return epk
