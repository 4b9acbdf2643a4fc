"""The overlap model (SPEC.md:376 recurrence) against SPEC.md's hand-evaluated examples."""
import json
import os

import pytest

from paper_2508_18572_b200.overlap import pipeline_recurrence

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pipeline_recurrence.json")))


@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["cite"][:14] for c in GOLD["cases"]])
def test_recurrence_golden(case):
    comp, wall, stall = pipeline_recurrence(case["t_load"], case["t_comp"])
    assert wall == case["wall"]
    assert stall == case["stall"]
    if "comp_finish" in case:
        assert comp == case["comp_finish"]


def test_recurrence_bounds():
    # wall is at least the total load plus the last layer's compute, and at least all compute
    t_load, t_comp = [3, 1, 4, 1, 5], [2, 7, 1, 8, 2]
    _, wall, stall = pipeline_recurrence(t_load, t_comp)
    assert wall >= sum(t_load) + t_comp[-1]
    assert wall >= t_load[0] + sum(t_comp)
    assert wall <= sum(t_load) + sum(t_comp)
    assert stall >= 0
