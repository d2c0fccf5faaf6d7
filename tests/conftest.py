import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through the C-ABI library)")
    config.addinivalue_line("markers", "slow: long CPU test (still part of the default run)")


def _group_fullsize_by_config(items):
    """tests/test_gpu_fullsize.py: run each BASELINE config's lockstep and gates tests back
    to back, so that its full-size instance (kept one at a time in host memory) is generated
    once instead of twice (huge ~40 s, multi ~60 s).  Only the order inside that module's
    parametrized block changes."""
    order = {"medium": 0, "huge": 1, "multi": 2}
    pos = [i for i, it in enumerate(items)
           if it.nodeid.startswith("tests/test_gpu_fullsize.py") and getattr(it, "callspec", None) is not None
           and it.callspec.params.get("name") in order]
    grouped = sorted((items[i] for i in pos), key=lambda it: order[it.callspec.params["name"]])   # stable
    for i, it in zip(pos, grouped):
        items[i] = it


def pytest_collection_modifyitems(config, items):
    _group_fullsize_by_config(items)
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
