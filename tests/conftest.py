import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: long-running")


def _gpu_count() -> int:
    try:
        from paper_1905_01549_b200 import cgvk

        return cgvk.device_count()
    except Exception:
        return 0


def pytest_collection_modifyitems(config, items):
    if any("gpu" in item.keywords for item in items) and _gpu_count() == 0:
        skip = pytest.mark.skip(reason="no CUDA device visible")
        for item in items:
            if "gpu" in item.keywords:
                item.add_marker(skip)
