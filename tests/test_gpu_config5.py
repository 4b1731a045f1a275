"""configs[4] at full size against the REFERENCE itself: matmul_chain(1415) +
matmul-merge-shared-lhs, k_multi=1, k_max=1 (10,009,713 e-nodes, 6,008,093
classes).  tests/golden/config5_golden_n1415.json was made by
tests/golden/make_model_golden.py running /root/reference (605 s, one core):
sha256 of the iteration's dump() and filter list, the non-time stats, the cost
vector, the greedy selection and total.  The device must reproduce all of them."""

import json
import os

import pytest

from paper_2101_01332_b200 import bench_graphs
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.tensor_lang import build_egraph, emit_graph, make_single_rooted, parse_graph

import make_model_golden as MG

pytestmark = pytest.mark.gpu

CASE = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config5_golden_n1415.json")))


def test_config5_matches_reference():
    text = emit_graph(bench_graphs.matmul_chain(CASE["n"]))
    assert MG.sha(text) == CASE["graph_sha"]
    g = make_single_rooted(parse_graph(text))
    rules = [r for r in default_rules() if r.name in CASE["rules"]]
    eg, _ = build_egraph(g)
    filt, rep = saturate(eg, rules, ExploreLimits(n_max=CASE["n_max"], k_max=CASE["k_max"], k_multi=CASE["k_multi"]),
                         "efficient", filt=set())
    assert {k: v for k, v in rep.to_stats().items() if "time" not in k} == CASE["stats"]
    it = CASE["iterations"][-1]
    assert (eg.num_nodes, eg.num_classes) == (it["nodes"], it["classes"])
    assert MG.sha(eg.dump()) == it["dump_sha"] == CASE["final_dump_sha"]
    assert MG.sha(MG.filt_text(filt)) == CASE["final_filt_sha"]
    costs = egraph_costs(eg, CostModel())
    assert MG.sha(MG.costs_text({int(k): costs[k] for k in costs})) == CASE["costs_sha"]
    res = greedy_extract(eg, costs, filt)
    assert len(res.selection) == CASE["selection_size"]
    assert MG.sha(MG.selection_text(res.selection)) == CASE["selection_sha"]
    assert res.total_cost == pytest.approx(CASE["total"], rel=1e-9)
