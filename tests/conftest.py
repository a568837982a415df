import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built librsk")
    config.addinivalue_line("markers", "slow: longer CPU test")


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def rsk():
    """The CUDA product path (fails loudly if the extension is missing on a GPU box)."""
    if not cuda_available():
        pytest.skip("no CUDA device")
    import paper_2306_15049_b200 as pkg
    return pkg
