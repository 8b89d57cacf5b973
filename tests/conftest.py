import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu(n): needs at least n CUDA devices")


def _gpu_count():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:  # pragma: no cover
        return 0


def pytest_collection_modifyitems(config, items):
    n = None
    for item in items:
        m = item.get_closest_marker("multigpu")
        if m is None:
            continue
        if n is None:
            n = _gpu_count()
        need = m.args[0] if m.args else 2
        if n < need:
            item.add_marker(pytest.mark.skip(reason=f"needs {need} GPUs, have {n}"))
