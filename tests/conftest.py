import gzip
import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name: str):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rb") as fh:
            return json.loads(fh.read())
    with open(path) as fh:
        return json.load(fh)


def terms_in(rows):
    """[[i, j, "c"], ...] -> {(i, j): c}"""
    return {(int(i), int(j)): int(c) for i, j, c in rows}


def ints_in(xs):
    return [int(x) for x in xs]


@pytest.fixture(scope="session")
def small():
    return load_golden("small.json")


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.build()
    return oracle
