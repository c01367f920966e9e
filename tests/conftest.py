"""Test configuration: registers the `gpu` marker and puts the repo root
(package + oracle/) on sys.path."""
import os
import sys

# deterministic cuBLAS workspaces, so tests may enable torch's deterministic
# algorithms (must be set before the first cuBLAS handle is created)
os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
