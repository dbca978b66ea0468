import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF = "/root/reference/proj"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def native():
    """Build (incrementally) and load the product libraries."""
    from paper_2503_01890_b200 import build
    build.build()
    from paper_2503_01890_b200 import _native
    return _native.lib()


@pytest.fixture(scope="session")
def oracle_built():
    import subprocess
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "adam"], check=True, capture_output=True)
    return True


def have_reference() -> bool:
    return os.path.isdir(os.path.join(REF, "core", "src"))


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
