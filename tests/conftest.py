import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

PRODUCT_LIB = os.path.join(ROOT, "paper_2512_20953_b200", "libhetplan_b200.so")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: longer CPU-side checks")


@pytest.fixture(scope="session")
def oracle():
    from oracle.binding import HPO_LIB, Oracle
    if not os.path.exists(HPO_LIB):
        pytest.skip("oracle not built (python -c 'import __graft_entry__ as g; g.build()')")
    return Oracle()


@pytest.fixture(scope="session")
def ref_lib():
    from oracle.binding import REF_LIB
    from paper_2512_20953_b200.capi import HetplanLib
    if not os.path.exists(REF_LIB):
        pytest.skip("reference library not built (oracle/_ref)")
    return HetplanLib(REF_LIB)


@pytest.fixture(scope="session")
def product_lib():
    from paper_2512_20953_b200.capi import HetplanLib
    if not os.path.exists(PRODUCT_LIB):
        pytest.fail("product library missing: build() must run before the tests")
    return HetplanLib(PRODUCT_LIB)


@pytest.fixture(scope="session")
def engine():
    from paper_2512_20953_b200.engine import Engine
    return Engine()


@pytest.fixture(scope="session")
def golden_plans():
    import json
    with open(os.path.join(GOLDEN, "plans.json")) as f:
        return {r["name"]: r for r in json.load(f)}


@pytest.fixture(scope="session")
def golden_grouping():
    import json
    with open(os.path.join(GOLDEN, "grouping.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_partition():
    import json
    with open(os.path.join(GOLDEN, "partition.json")) as f:
        return json.load(f)
