import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
# Every prune in the test process takes the fused cluster kernel whatever the batch (the library routes small
# per-token batches to the three separate kernels by default — covered by a subprocess test in
# test_kernels_gpu.py); the fused-vs-separate comparisons then exercise both paths on every shape.
os.environ.setdefault("QVK_PRUNE_FUSED_MIN_SEGS", "0")
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) — run with -m gpu on the GPU box")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return torch.device("cuda:0")
