from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_cases():
    with open(os.path.join(GOLDEN, "cases.json")) as f:
        return json.load(f)


_ARRAYS = None


def golden_arrays():
    global _ARRAYS
    if _ARRAYS is None:
        _ARRAYS = dict(np.load(os.path.join(GOLDEN, "tensors.npz")))
    return _ARRAYS


def case_tensors(case):
    a = golden_arrays()
    n = case["name"]
    ws = [a[f"{n}/w{j}"] for j in range(case["n_weights"])]
    dws = [a[f"{n}/dw{j}"] for j in range(case["n_weights"])]
    return a[f"{n}/x"], ws, a[f"{n}/up"], a[f"{n}/y"], a[f"{n}/y_staged"], dws


CASES = load_cases()
CASE_IDS = [c["name"] for c in CASES]


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")
