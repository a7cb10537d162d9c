import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """Make sure libadatopk.so exists (nvcc cross-compiles without a GPU)."""
    from paper_2410_12707_b200 import build

    if not build.LIB.exists():
        build.build()
    yield


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected but no CUDA device is visible (the AdaTopK path has no CPU fallback)")
    return torch.device("cuda", 0)
