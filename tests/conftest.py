import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


GOLDEN = os.path.join(REPO, "tests", "golden")


def load_golden(name):
    import numpy as np

    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def golden_pencil(g):
    n = int(g["n"])
    a = (g["a_rp"], g["a_ci"], g["a_v"])
    b = (g["b_rp"], g["b_ci"], g["b_v"]) if "b_rp" in g else None
    return (n, a, b)


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle

    return oracle.Oracle()
