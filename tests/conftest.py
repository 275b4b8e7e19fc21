import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU sweep")


@pytest.fixture(scope="session")
def ref():
    from _oracle import ref as _r
    return _r()


@pytest.fixture(scope="session")
def ora():
    from _oracle import ora as _o
    return _o()


@pytest.fixture(scope="session")
def ss():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    from paper_2603_20481_b200 import specsense
    return specsense
