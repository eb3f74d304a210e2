import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through libfmap_cuda")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    import oracle as o
    if not o.LIB.exists():
        o.build()
    return o


@pytest.fixture(scope="session")
def fm():
    """The product package; on a GPU box the CUDA library must load (no fallback)."""
    import paper_2604_10377_b200 as pkg
    pkg.load()
    return pkg


@pytest.fixture(scope="session")
def cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device (no CPU fallback)"
    return torch.device("cuda", 0)
