import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


@pytest.fixture(scope="session")
def golden_meta():
    with open(os.path.join(GOLDEN, "primitives.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_prims():
    return dict(np.load(os.path.join(GOLDEN, "primitives.npz")))


@pytest.fixture(scope="session")
def golden_loops():
    return dict(np.load(os.path.join(GOLDEN, "node_loops.npz")))


@pytest.fixture(scope="session")
def golden_pulls():
    return dict(np.load(os.path.join(GOLDEN, "pull_loops.npz")))


@pytest.fixture(scope="session")
def golden_config1():
    return dict(np.load(os.path.join(GOLDEN, "config1.npz")))
