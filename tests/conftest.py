import os
import sys

# The golden vectors were generated with single-threaded OpenBLAS; the oracle
# reproduces them bitwise only with the same summation order.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
try:  # numpy may already be loaded by a plugin: clamp the live BLAS pool too
    from threadpoolctl import threadpool_limits

    _BLAS_LIMIT = threadpool_limits(limits=1, user_api="blas")
except Exception:  # pragma: no cover
    _BLAS_LIMIT = None

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: long CPU oracle runs")


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
