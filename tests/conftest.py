"""Shared test setup: registers the ``gpu`` marker, makes the repo root
importable (package, ``oracle/`` checker) and loads golden fixtures."""

import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for _p in (ROOT, TESTS):
    if _p not in sys.path:
        sys.path.insert(0, _p)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built "
                            "libgstab_sm100a.so")


def load_golden(name):
    with gzip.open(os.path.join(GOLDEN, name), "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_shots():
    return load_golden("shots.json.gz")


@pytest.fixture(scope="session")
def golden_states():
    return load_golden("states.json.gz")


@pytest.fixture(scope="session")
def golden_counters():
    return load_golden("counters.json.gz")


@pytest.fixture(scope="session")
def golden_rng():
    return load_golden("rng.json.gz")
