import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(scope="session")
def gk():
    """The product library, built in-tree (nvcc) and loaded; needs a CUDA device."""
    import torch

    import paper_2103_14978_b200 as m
    from paper_2103_14978_b200 import _build
    _build.build()
    m.load_library()
    assert torch.cuda.is_available(), "GPU test without a CUDA device"
    return m
