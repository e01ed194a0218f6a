import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    """Golden vectors made by tests/golden/make_golden.py from the real reference."""
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        data = {k: z[k] for k in z.files}
    cases = {}
    for key, val in data.items():
        case, field = key.split("/", 1)
        cases.setdefault(case, {})[field] = val
    return cases


@pytest.fixture(scope="session")
def golden():
    return load_golden


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
