import os
import sys

# before torch creates a CUDA context (spawned rank processes inherit it): one
# hardware queue per stream, see INTEGRATION.md
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under `pytest -m gpu` on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


def n_gpus() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


@pytest.fixture
def need_gpus():
    def _need(n):
        if n_gpus() < n:
            pytest.skip(f"needs {n} GPUs, have {n_gpus()}")
    return _need
