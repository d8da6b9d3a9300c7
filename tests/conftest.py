import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def kats():
    with open(os.path.join(GOLDEN, "kats.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_layers():
    return dict(np.load(os.path.join(GOLDEN, "layers.npz")))


@pytest.fixture(scope="session")
def golden_terrain():
    return dict(np.load(os.path.join(GOLDEN, "terrain.npz")))


@pytest.fixture(scope="session")
def golden_rl():
    return dict(np.load(os.path.join(GOLDEN, "rl.npz")))


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O
    return O.port()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O
    R = O.ref()
    if R is None:
        pytest.skip("reference not built here (oracle/_ref); golden fixtures cover the port")
    return R


def layer_cases(golden_layers):
    names = sorted({k.split("_")[0] for k in golden_layers})
    out = []
    for n in names:
        out.append({k[len(n) + 1:]: v for k, v in golden_layers.items() if k.startswith(n + "_")})
    return out
