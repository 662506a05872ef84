import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "reference: needs /root/reference (this container only)")


def pytest_collection_modifyitems(config, items):
    from refcompat import reference_available
    if reference_available():
        return
    skip = pytest.mark.skip(reason="/root/reference is not present (GPU box)")
    for item in items:
        if "reference" in item.keywords:
            item.add_marker(skip)
