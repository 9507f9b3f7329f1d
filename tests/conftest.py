import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def gpu_lib():
    """The CUDA path; fails loudly (never falls back) when the extension or GPU is missing."""
    import torch
    assert torch.cuda.is_available(), "GPU test run without a GPU"
    from paper_1008_3699_b200 import binding
    binding.load()
    return binding
