import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)

TREE_CASES = sorted(
    f[len("tree_"):-len(".npz")] for f in os.listdir(GOLDEN) if f.startswith("tree_")
)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size configurations")


def load_case(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"tree_{name}.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_cases():
    return {name: load_case(name) for name in TREE_CASES}


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
