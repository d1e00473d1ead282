"""End-to-end parity through the drop-in C ABI on the GPU: hp_plan_compute of
libhetplan_b200.so returns byte-identical plan JSON (or the identical status
and error text) to the reference library on every catalog case (BASELINE
configs, reference fixtures, acceptance clusters, every planner option)."""
import pytest

from paper_2512_20953_b200 import cases
from paper_2512_20953_b200.capi import HetplanError

pytestmark = pytest.mark.gpu

CASES = cases.plan_cases()


def _plan(lib, case):
    try:
        return 0, lib.plan_json(case.cluster, case.model, case.max_layers, case.options,
                                case.base_seconds)
    except HetplanError as e:
        return e.status, e.message


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_plan_matches_golden(product_lib, golden_plans, case):
    g = golden_plans[case.name]
    status, out = _plan(product_lib, case)
    assert status == g["status"], out
    if status == 0:
        assert out == g["json"]
    else:
        assert out == g["error"]


def test_plan_matches_live_reference(product_lib, ref_lib):
    for case in cases.plan_cases(include_heavy=False):
        assert _plan(product_lib, case) == _plan(ref_lib, case), case.name


def test_plan_is_deterministic(product_lib):
    case = [c for c in CASES if c.name == "accept-c10-24gpu"][0]
    assert _plan(product_lib, case) == _plan(product_lib, case)
