import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the CUDA path")


@pytest.fixture(scope="session")
def oracle():
    from oracle import model
    model.build()
    return model


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        return cache[name]
    return load


def counter_keys(seed, n):
    """Uniform distinct 64-bit keys (the reference's counter_stream,
    workloads.py:23-26, restated in paper_2212_09005_b200.workloads)."""
    from paper_2212_09005_b200.workloads import counter_stream
    return counter_stream(seed, 0x5851F42D4C957F2D, n)
