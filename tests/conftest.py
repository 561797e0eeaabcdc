import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _ensure_library():
    """Build libtdes_b200.so if it is missing (nvcc cross-compiles without a GPU)."""
    lib = os.path.join(ROOT, "paper_2007_10752_b200", "libtdes_b200.so")
    if not os.path.exists(lib):
        import __graft_entry__
        __graft_entry__.build_library()


def pytest_configure(config):
    _ensure_library()
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_kat():
    """Parse tests/golden/des_kat.txt into a list of (kind, fields, citation)."""
    rows = []
    with open(os.path.join(ROOT, "tests", "golden", "des_kat.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            parts = line.split()
            rows.append((parts[0], parts[1:-1], parts[-1]))
    return rows


@pytest.fixture(scope="session")
def kat_rows():
    return load_kat()


def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
