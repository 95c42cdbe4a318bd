import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running statistical or full-size case")
    config.addinivalue_line("markers", "sanitize: compute-sanitizer run over the concurrency-heavy paths")


def pytest_collection_modifyitems(config, items):
    # GPU tests fail loudly (not skip) when selected without a GPU: a silent skip
    # would hide a missing CUDA path.  They are only selected with -m gpu.
    pass
