import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: long-running case")


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    g = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(g, "golden.json")) as f:
        meta = json.load(f)
    return {
        "meta": meta,
        "rng": dict(np.load(os.path.join(g, "rng.npz"))),
        "sketch": dict(np.load(os.path.join(g, "sketch.npz"))),
        "pipeline": dict(np.load(os.path.join(g, "pipeline.npz"))),
        "gradient": dict(np.load(os.path.join(g, "gradient.npz"))),
    }
