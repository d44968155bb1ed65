import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box via gpurun)")


@pytest.fixture(scope="session")
def lz():
    import paper_2406_10707_b200 as L
    return L


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    return O


@pytest.fixture(scope="session")
def fixtures():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "ref_fixtures.json")) as f:
        return json.load(f)["cases"]


@pytest.fixture(scope="session")
def cases():
    from cases import all_cases
    return {w.name: (w, thr) for w, thr in all_cases()}
