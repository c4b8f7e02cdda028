import glob
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


@pytest.fixture(scope="session")
def ref():
    from oracle.bindings import Ref
    return Ref()


@pytest.fixture(scope="session")
def port():
    from oracle.bindings import Port
    return Port()


@pytest.fixture(scope="session")
def kat():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


def golden_names():
    return sorted(os.path.basename(p)[4:-5] for p in glob.glob(os.path.join(GOLDEN, "idx_*.ptrh")))


def load_golden(name):
    with open(os.path.join(GOLDEN, f"idx_{name}.ptrh"), "rb") as f:
        ptrh = f.read()
    with open(os.path.join(GOLDEN, f"idx_{name}.json")) as f:
        rec = json.load(f)
    return ptrh, rec
