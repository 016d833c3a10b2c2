"""Test-session setup: GPU marker, repo on sys.path, BLAS pinned to 1 thread
(the oracle's numpy matmuls must be bit-reproducible run to run)."""

import os
import sys

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import pytest  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


def pytest_collection_modifyitems(config, items):
    for item in items:
        if "multigpu" in item.keywords and "gpu" not in item.keywords:
            item.add_marker(pytest.mark.gpu)


@pytest.fixture(scope="session")
def P():
    """The product package (GPU tests)."""
    import paper_1811_03619_b200 as pkg
    return pkg
