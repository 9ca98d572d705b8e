"""Shared pytest configuration.

Markers:
  gpu -- needs a CUDA device (B200); the driver runs `pytest -m gpu` on the box
         and `pytest -m "not gpu"` here (no GPU).
"""

import gzip
import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rb") as f:
            return json.loads(f.read())
    with open(path) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_sorts():
    return load_golden("sorts.json.gz")


@pytest.fixture(scope="session")
def golden_profiles():
    return load_golden("profiles.json.gz")


@pytest.fixture(scope="session")
def golden_powers():
    return load_golden("powers.json.gz")


@pytest.fixture(scope="session")
def golden_cfg_full():
    return load_golden("cfg_full.json")
