import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """Build libcronus_b200.so in-tree if it is missing (the GPU box gets the prebuilt
    library with the snapshot; objects are not shipped, so never rebuild there)."""
    from paper_2509_17357_b200 import build
    if not os.path.exists(build.LIB) or os.path.isdir(build.BUILD):
        build.build()
    yield


CONFIG_DIR = os.path.join(ROOT, "tests", "golden", "configs")


def load_cfg(name):
    with open(os.path.join(CONFIG_DIR, name + ".cfg")) as f:
        return f.read()
