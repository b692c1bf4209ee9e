"""Shared test setup.

Markers: `gpu` = needs a B200 (run with -m gpu on the GPU box); everything
else runs on CPU.  Golden fixtures come from tests/golden/make_golden.py,
which ran the reference itself in the build container.
"""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running case")


def load_golden(name):
    meta = json.load(open(os.path.join(GOLDEN, name + ".json")))
    path = os.path.join(GOLDEN, name + ".npz")
    arrays = np.load(path) if os.path.exists(path) else None
    return meta, arrays


@pytest.fixture(scope="session")
def golden():
    return load_golden


@pytest.fixture(scope="session")
def oracle():
    from oracle import port
    port.lib()
    return port
