"""GPU parity on the authored model graphs against the REFERENCE itself
(tests/golden/model_golden.json, made by tests/golden/make_model_golden.py
running /root/reference): after EVERY iteration the sha256 of dump() and of
the sorted filter list, then the non-time stats, the cost vector (every fp64
value, id order), the greedy selection and total.  The oracle is not involved:
these pin the device engine to the reference directly, at the bench configs
(BERT to its 50k node limit, the k_multi=2 graphs to saturation)."""

import json
import os

import pytest

from paper_2101_01332_b200 import models
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.tensor_lang import build_egraph, emit_graph, make_single_rooted, parse_graph

import make_model_golden as MG

pytestmark = pytest.mark.gpu

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "model_golden.json")))


@pytest.mark.parametrize("case", CASES, ids=[c["id"] for c in CASES])
def test_model_graph_every_iteration_matches_reference(case):
    text = emit_graph(models.MODELS[case["model"]]())
    assert MG.sha(text) == case["graph_sha"], "authored graph changed since the fixture was made"
    g = make_single_rooted(parse_graph(text))
    rules = list(default_rules())
    eg, _ = build_egraph(g)
    filt = set()
    its = case["iterations"]
    for i, snap in enumerate(its):
        lim = ExploreLimits(n_max=case["n_max"], k_max=1, k_multi=1 if i < case["k_multi"] else 0)
        filt, rep = saturate(eg, rules, lim, "efficient", filt=filt)
        assert (eg.num_nodes, eg.num_classes) == (snap["nodes"], snap["classes"]), f"iteration {i}"
        assert MG.sha(eg.dump()) == snap["dump_sha"], f"iteration {i}"
        assert MG.sha(MG.filt_text(filt)) == snap["filt_sha"], f"iteration {i}"
    costs = egraph_costs(eg, CostModel())
    assert MG.sha(MG.costs_text({int(k): costs[k] for k in costs})) == case["costs_sha"]
    res = greedy_extract(eg, costs, filt)
    assert len(res.selection) == case["selection_size"]
    assert MG.sha(MG.selection_text(res.selection)) == case["selection_sha"]
    assert res.total_cost == pytest.approx(case["total"], rel=1e-9)


@pytest.mark.parametrize("case", CASES, ids=[c["id"] for c in CASES])
def test_model_graph_one_shot_matches_reference(case):
    """The same search in one explore-style saturate call: final state and stats."""
    g = make_single_rooted(parse_graph(emit_graph(models.MODELS[case["model"]]())))
    eg, _ = build_egraph(g)
    filt, rep = saturate(eg, list(default_rules()),
                         ExploreLimits(n_max=case["n_max"], k_max=case["k_max"], k_multi=case["k_multi"]),
                         "efficient", filt=set())
    assert {k: v for k, v in rep.to_stats().items() if "time" not in k} == case["stats"]
    assert MG.sha(eg.dump()) == case["final_dump_sha"]
    assert MG.sha(MG.filt_text(filt)) == case["final_filt_sha"]
