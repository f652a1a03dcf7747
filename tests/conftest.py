"""Shared pytest setup.

* ``gpu`` marks tests that need a B200 (run by the driver with ``-m gpu``).
* The CPU oracle (``oracle/``) is test infrastructure: tests load it as the
  checker; the product package never imports it.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


def _ensure_oracle():
    import oracle as O
    if not os.path.exists(O.PORT_LIB):
        import subprocess
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True,
                       capture_output=True)
    return O


@pytest.fixture(scope="session")
def O():
    return _ensure_oracle()


@pytest.fixture(scope="session")
def port(O):
    return O.Oracle("port")


@pytest.fixture(scope="session")
def ref(O):
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return O.Oracle("reference")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    return load


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_03275_b200 import ops
    ops.context()
    return torch.device("cuda")
