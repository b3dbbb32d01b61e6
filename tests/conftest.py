import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")

# tests/reference_backend/ holds the INTEGRATION.md stub and a reference-side
# test module; they import `tsetlinkit` and only run inside the patched
# reference copy tools/run_reference_suite.py builds (via
# tests/test_reference_suite_b200.py), never from this tree.
collect_ignore = ["reference_backend"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtmb200.so")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    o.build()
    return o


@pytest.fixture(scope="session")
def gpu():
    """The product package on a CUDA device; fails loudly without one."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu-marked test run without a CUDA device")
    import paper_2405_04212_b200 as tmb
    tmb.runtime.require_device()
    return tmb
