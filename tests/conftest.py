import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(TESTS, "golden")
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (run with -m gpu)")
    config.addinivalue_line("markers", "slow: large configs (minutes)")


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def small_golden():
    meta = json.load(open(os.path.join(GOLDEN, "small.json")))
    arrays = np.load(os.path.join(GOLDEN, "small.npz"))
    cases = []
    for c in meta["cases"]:
        d = {}
        for k, v in c.items():
            d[k] = arrays[v] if isinstance(v, str) and v.startswith("c") and v in arrays.files else v
        cases.append(d)
    return {"cases": cases, "kat": meta["kat"]}


@pytest.fixture(scope="session")
def configs_golden():
    path = os.path.join(GOLDEN, "configs.json")
    if not os.path.exists(path):
        pytest.skip("configs.json not generated")
    return json.load(open(path))


@pytest.fixture(scope="session")
def gpu():
    if not gpu_available():
        pytest.skip("no CUDA device")
    import torch

    return torch.device("cuda", 0)
