import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); parity tests through the C-ABI")


@pytest.fixture(scope="session")
def oracle():
    import oracle_ffi

    oracle_ffi.build()
    return oracle_ffi


@pytest.fixture(scope="session")
def vd():
    import paper_2604_04310_b200 as vd

    return vd


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test collected but no CUDA device is visible")
    return torch.device("cuda", 0)
