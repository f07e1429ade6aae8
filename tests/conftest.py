import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs on the GPU box")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def load_small(idx):
    return dict(np.load(os.path.join(GOLDEN, f"small_{idx:02d}.npz")))


SMALL_IDS = sorted(int(f[6:8]) for f in os.listdir(GOLDEN) if f.startswith("small_") and f.endswith(".npz"))
