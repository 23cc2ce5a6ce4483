import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    if not os.path.exists(O.ORACLE_SO):
        O.build()
    return O


@pytest.fixture(scope="session")
def ctx():
    import paper_1012_2273_b200 as P
    c = P.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="session")
def golden_small():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "ref_small.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_big():
    import json
    p = os.path.join(ROOT, "tests", "golden", "ref_big.json")
    if not os.path.exists(p):
        pytest.skip("ref_big.json not generated")
    with open(p) as f:
        return json.load(f)
