import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libveckm.so")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


GOLDEN_CASES = [
    "small_d16", "cfg1_20k", "r20_12k", "dense_asym",
    "edge_single", "edge_pair_same_px", "edge_corner", "edge_far_corner",
    "edge_unsorted_dups", "edge_t_offset", "edge_bias_only",
]


@pytest.fixture(params=GOLDEN_CASES)
def golden_case(request):
    g = load_golden(request.param)
    g["name"] = request.param
    return g


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)
