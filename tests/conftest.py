import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gmr():
    """The CUDA product path; fails loudly (never falls back) without it."""
    if not cuda_available():
        pytest.fail("gpu test collected on a machine without CUDA")
    import paper_2602_14493_b200 as pkg
    pkg.lib.load()
    return pkg
