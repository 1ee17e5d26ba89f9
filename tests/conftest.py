import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: longer-running case")


@pytest.fixture(scope="session")
def phi_golden():
    with open(os.path.join(GOLDEN, "phi_vectors.json")) as f:
        index = json.load(f)
    data = np.load(os.path.join(GOLDEN, "phi_vectors.npz"))
    return index, data


@pytest.fixture(scope="session")
def mgrit_golden():
    with open(os.path.join(GOLDEN, "mgrit_cases.json")) as f:
        meta = json.load(f)
    data = np.load(os.path.join(GOLDEN, "mgrit_cases.npz"))
    return {m["name"]: m for m in meta}, data


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def sw_golden():
    with open(os.path.join(GOLDEN, "sw_vectors.json")) as f:
        index = json.load(f)
    data = np.load(os.path.join(GOLDEN, "sw_vectors.npz"))
    return index, data


@pytest.fixture(scope="session")
def sw_mgrit_golden():
    with open(os.path.join(GOLDEN, "sw_mgrit_cases.json")) as f:
        meta = json.load(f)
    data = np.load(os.path.join(GOLDEN, "sw_mgrit_cases.npz"))
    return {m["name"]: m for m in meta}, data


@pytest.fixture(scope="session")
def euler_golden():
    with open(os.path.join(GOLDEN, "euler_vectors.json")) as f:
        index = json.load(f)
    data = np.load(os.path.join(GOLDEN, "euler_vectors.npz"))
    return index, data
