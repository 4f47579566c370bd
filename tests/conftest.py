"""Shared fixtures.  `-m "not gpu"` runs the oracle / host-logic / ABI suite
on CPU; `-m gpu` runs the parity tests through the C-ABI on a B200."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running")


def have_ref() -> bool:
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libgwref.so"))


@pytest.fixture(scope="session")
def port():
    from oracle.bindings import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    if not have_ref():
        pytest.skip("reference build (oracle/_ref) not present")
    from oracle.bindings import Oracle
    return Oracle("reference")


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    from paper_2205_08115_b200 import abi
    abi.load()
    return torch.device("cuda:0")
