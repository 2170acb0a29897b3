"""pytest configuration: markers, in-tree native builds, shared fixtures."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long CPU test (full-size configs)")


def _make(target, artefact):
    path = os.path.join(ROOT, artefact)
    src_newer = False
    if os.path.exists(path):
        return path
    subprocess.run(["make", "-C", ROOT, target], check=True, capture_output=not src_newer)
    return path


@pytest.fixture(scope="session", autouse=True)
def native_host_libs():
    """gen/ and oracle/ are plain C: build them if missing (seconds)."""
    _make("gen", "gen/libgcgen.so")
    _make("oracle", "oracle/liboracle.so")
    yield


@pytest.fixture(scope="session")
def gc_lib_path():
    return _make("gc", "paper_1708_06866_b200/libgc.so")
