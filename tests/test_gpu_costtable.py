"""Device cost-TABLE mode (egraph_costs with a load_cost_table model,
reference cost.py:135-196, 225-247) against the reference's own vectors
(tests/golden/costtable_golden.json, made by make_costtable_golden.py):
signature keys are rendered on the device and looked up in the table, misses
fall back to the synthetic formula; strict tables raise UnknownSignature with
the reference's message."""

import json
import os

import pytest

import cases
from paper_2101_01332_b200 import bench_graphs, tensor_lang
from paper_2101_01332_b200.cost import egraph_costs, load_cost_table
from paper_2101_01332_b200.errors import NoFiniteExtraction, UnknownSignature
from paper_2101_01332_b200.explorer import ExploreLimits, explore
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.rules import default_rules

pytestmark = pytest.mark.gpu

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "costtable_golden.json")))


@pytest.mark.parametrize("case", CASES, ids=[c["id"] for c in CASES])
def test_cost_table_vector_matches_reference(case):
    g = cases.build_graph(bench_graphs, tensor_lang, case["graph"])
    eg, filt, _ = explore(g, list(default_rules()), ExploreLimits(k_multi=case["k_multi"], k_max=case["k_max"]))
    model = load_cost_table(case["table"])
    costs = egraph_costs(eg, model)
    assert {str(k): costs[k] for k in costs} == case["costs"]
    if "error" in case["greedy"]:
        with pytest.raises(NoFiniteExtraction):
            greedy_extract(eg, costs, filt)
    else:
        res = greedy_extract(eg, costs, filt)
        assert {str(k): v for k, v in sorted(res.selection.items())} == case["greedy"]["selection"]
        assert res.total_cost == pytest.approx(case["greedy"]["total"], rel=1e-9)
    strict = load_cost_table(case["table"], strict=True)
    if case["strict_error"] is None:
        egraph_costs(eg, strict)
    else:
        with pytest.raises(UnknownSignature) as ei:
            egraph_costs(eg, strict)
        assert str(ei.value) == case["strict_error"]
