import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


SMALL_CASES = ["small_cube_p5", "small_cube_p6", "small_brick_p6", "small_brick_p8",
               "small_brick_p7", "small_cube_p4", "small_single"]
TRI_CASES = [("tri_skew_p8", (64, 64, 80)), ("tri_skew_p6", (48, 48, 60)),
             ("tri_flex_p7", (44, 48, 52))]


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")
