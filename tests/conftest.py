import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: large-size GPU case")


def pytest_collection_modifyitems(config, items):
    # GPU tests fail loudly (never skip silently) when selected with -m gpu
    # on a box without a device; on CPU runs they are deselected by -m.
    pass
