import os
import sys
from pathlib import Path

import pytest

# Rank-mode patch lanes wait on peer signals with stream memory operations;
# several ranks sharing one GPU in one process need more hardware queues than
# the default 8, or a blocked lane can stall an unrelated stream behind it.
# Must be set before the CUDA context exists (see paper_2405_14430_b200
# runtime: rank-mode lanes need >= 16).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200, sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running case")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
