import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a engine)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def engine():
    import paper_2407_20713_b200 as pkg

    eng = pkg.Engine(0)
    yield eng
    eng.close()


@pytest.fixture(scope="session")
def ref():
    from oracles import Ref, have_ref

    if not have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Ref()


@pytest.fixture(scope="session")
def orc():
    from oracles import Restate, have_restate

    if not have_restate():
        pytest.skip("oracle restatement not built")
    return Restate()


@pytest.fixture(scope="session")
def eq_surface():
    import paper_2407_20713_b200 as pkg

    return pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurostoxx50.csv"))


@pytest.fixture(scope="session")
def fx_surface():
    import paper_2407_20713_b200 as pkg

    return pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurusd.csv"))
