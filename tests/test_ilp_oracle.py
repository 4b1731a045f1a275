"""ILP model build: the CPU oracle (oracle.tsat_oracle.oracle_build_ilp) against
the reference's own reachable classes and LP text (tests/golden/ilp_golden.json,
made by tests/golden/make_ilp_golden.py).  CPU only; the LP text is formatted
with the host export_lp, which needs no GPU."""

import json
import os

import pytest

import cases
from oracle import tsat_oracle as O
from paper_2101_01332_b200 import bench_graphs, tensor_lang
from paper_2101_01332_b200.cost import CostModel
from paper_2101_01332_b200.extract import ILPModel, export_lp
from paper_2101_01332_b200.rules import default_rules

HERE = os.path.join(os.path.dirname(__file__), "golden")
ILP = json.load(open(os.path.join(HERE, "ilp_golden.json")))
BY_ID = {c[0]: c for c in cases.EXPLORE_CASES}


def oracle_case(cid):
    _, gspec, names, limits, mode, self_pairs = BY_ID[cid]
    g = cases.build_graph(bench_graphs, tensor_lang, gspec)
    rules = cases.select_rules(default_rules(), names)
    eg, filt, _ = O.oracle_explore(g, rules, filter_mode=mode, allow_self_pairs=self_pairs, **limits)
    return eg, filt, O.oracle_costs(eg, CostModel())


def as_model(m: dict, with_cycle: bool, topo: str) -> ILPModel:
    nx = sum(1 for n in m["var_names"] if n.startswith("x_"))
    t_of_class = {c: nx + i for i, c in enumerate(m["classes"])} if with_cycle else {}
    return ILPModel(var_names=m["var_names"], objective=m["objective"], lb=m["lb"], ub=m["ub"],
                    binary_idx=list(range(nx)), integer_idx=list(t_of_class.values()) if topo == "int" else [],
                    rows=m["rows"], t_of_class=t_of_class, class_order=m["classes"], with_cycle=with_cycle,
                    topo=topo)


@pytest.mark.parametrize("rec", ILP, ids=[r["id"] for r in ILP])
def test_oracle_ilp_matches_reference(rec):
    eg, filt, costs = oracle_case(rec["id"])
    assert O.oracle_reachable_classes(eg, filt) == rec["reachable"]
    for v in rec["variants"]:
        m = O.oracle_build_ilp(eg, costs, filt, with_cycle=v["with_cycle"], topo=v["topo"])
        assert len(m["rows"]) == v["num_rows"]
        assert export_lp(as_model(m, v["with_cycle"], v["topo"])) == v["lp"], v["variant"]
