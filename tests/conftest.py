"""Shared pytest setup.

Markers: ``gpu`` — needs a B200 (run by the driver with ``-m gpu`` on the GPU box);
everything else runs on CPU here with ``-m "not gpu"``.

The CPU oracle (``oracle/``) is imported only by tests, never by the product.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    return oracle.ref()


@pytest.fixture(scope="session")
def golden_sweep():
    return np.load(os.path.join(GOLDEN, "sweep_golden.npz"))


@pytest.fixture(scope="session")
def golden_json():
    def load(name):
        with open(os.path.join(GOLDEN, name)) as f:
            return json.load(f)
    return load


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    from paper_2407_13096_b200.api import Context
    c = Context(0)
    yield c
    c.close()


@pytest.fixture(params=[0, 1], ids=["ffma", "tc"])
def engine(request, ctx):
    """Runs a predictor test on both engines: the FMA-pipe kernel (0) and the
    tcgen05 3xTF32 kernel (1); restores the default afterwards."""
    ctx.set_option("mlp_engine", request.param)
    yield request.param
    ctx.set_option("mlp_engine", 2)
