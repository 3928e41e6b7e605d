import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C ABI on cuda:0)")
    config.addinivalue_line("markers", "reference: imports the reference package (this container only)")
    config.addinivalue_line("markers", "slow: long-running")


def have_reference():
    return os.path.isdir(os.path.join(REF_SRC, "mgtrace"))


@pytest.fixture(scope="session")
def mgtrace_ref():
    if not have_reference():
        pytest.skip("reference package not present (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import mgtrace
    return mgtrace


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
