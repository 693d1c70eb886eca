import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


@pytest.fixture(scope="session")
def oracle():
    from _oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from _oracle import RefLib

    if not RefLib.available():
        pytest.skip("oracle/_ref (the compiled reference) is not built here")
    return RefLib()


@pytest.fixture(scope="session")
def ctx():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    from paper_2508_03984_b200 import Context

    return Context(0)
