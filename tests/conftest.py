import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_CUDA = _cuda()


def pytest_collection_modifyitems(config, items):
    if HAS_CUDA:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def unit_golden():
    return np.load(os.path.join(GOLDEN, "unit.npz"))


@pytest.fixture(scope="session")
def stepper_golden():
    arrays = np.load(os.path.join(GOLDEN, "steppers.npz"))
    with open(os.path.join(GOLDEN, "steppers.json")) as f:
        meta = json.load(f)
    return meta, arrays


@pytest.fixture(scope="session")
def config_golden():
    arrays = np.load(os.path.join(GOLDEN, "configs.npz"))
    with open(os.path.join(GOLDEN, "configs.json")) as f:
        meta = {m["tag"]: m for m in json.load(f)}
    return meta, arrays


def rel_l2(a, b):
    """||a - b||_2 / ||b||_2, scaled first so huge-but-finite states do not overflow."""
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    s = float(np.max(np.abs(b))) if b.size else 1.0
    s = s if s > 0 and np.isfinite(s) else 1.0
    return float(np.linalg.norm(a / s - b / s) / np.linalg.norm(b / s))


def rel_max(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(np.asarray(b))))
