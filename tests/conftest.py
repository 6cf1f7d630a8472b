"""Shared fixtures. `-m gpu` tests need a B200 and the in-tree libsfkv.so; everything else runs
on CPU. The CPU oracle (oracle/, test infrastructure) is built on demand here."""
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


@pytest.fixture(scope="session")
def oracle_api():
    import oracle_lib
    return oracle_lib.load()


@pytest.fixture(scope="session")
def gpu_api():
    import paper_2603_13605_b200 as pkg
    return pkg.api()
