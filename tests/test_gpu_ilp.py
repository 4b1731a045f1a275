"""GPU ILP path: the device model skeleton (csrc/ilp.cu through tsat_ilp_build)
against the reference's LP text and optimum (tests/golden/ilp_golden.json) and
against the CPU oracle on seeded graphs; the drop-in run_optimize with the
reference's default extractor.  Optimum: total within 1e-6 relative (the
reference's own branch-and-bound and HiGHS may pick different equal-cost
selections)."""

import json
import os
import random

import pytest

import cases
from oracle import tsat_oracle as O
from paper_2101_01332_b200 import bench_graphs, tensor_lang
from paper_2101_01332_b200.cli import RunConfig, run_optimize
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.errors import CyclicSelection
from paper_2101_01332_b200.explorer import ExploreLimits, explore
from paper_2101_01332_b200.extract import (build_ilp, export_lp, greedy_extract, parse_solution,
                                           reachable_classes, solve_ilp)
from paper_2101_01332_b200.rules import default_rules

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(__file__), "golden")
ILP = json.load(open(os.path.join(HERE, "ilp_golden.json")))
BY_ID = {c[0]: c for c in cases.EXPLORE_CASES}


def gpu_case(cid):
    _, gspec, names, limits, mode, self_pairs = BY_ID[cid]
    g = cases.build_graph(bench_graphs, tensor_lang, gspec)
    rules = cases.select_rules(default_rules(), names)
    eg, filt, _ = explore(g, rules, ExploreLimits(**limits), mode, allow_self_pairs=self_pairs)
    return eg, filt, egraph_costs(eg, CostModel())


@pytest.mark.parametrize("rec", ILP, ids=[r["id"] for r in ILP])
def test_ilp_model_and_optimum_match_reference(rec):
    eg, filt, costs = gpu_case(rec["id"])
    assert reachable_classes(eg, filt, eg.root) == rec["reachable"]
    for v in rec["variants"]:
        m = build_ilp(eg, costs, filt, with_cycle=v["with_cycle"], topo=v["topo"])
        assert m.num_vars == v["num_vars"]
        assert len(m.rows) == v["num_rows"]
        assert export_lp(m) == v["lp"], v["variant"]
        if "error" in v:
            # the reference's optimum was cyclic; HiGHS may land on another optimum
            try:
                solve_ilp(m, eg, 60.0)
            except CyclicSelection:
                pass
            continue
        r = solve_ilp(m, eg, 60.0)
        assert r.optimal
        assert r.total_cost == pytest.approx(v["total"], rel=1e-6)


@pytest.mark.parametrize("seed", range(6))
def test_ilp_rows_match_oracle_on_fuzz(seed):
    rng = random.Random(seed)
    name = rng.choice(["matmul-chain", "rnn-cell-stack", "conv-fanout", "inception-block"])
    g = bench_graphs.generate(name, rng.randint(1, 3), random.Random(seed))
    rules = default_rules()
    mode = rng.choice(["efficient", "none", "vanilla"])
    lim = dict(n_max=400, k_max=3, k_multi=1)
    eg, filt, _ = explore(g, rules, ExploreLimits(**lim), mode)
    oeg, ofilt, _ = O.oracle_explore(g, rules, filter_mode=mode, **lim)
    assert eg.dump() == oeg.dump()
    costs = egraph_costs(eg, CostModel())
    ocosts = O.oracle_costs(oeg, CostModel())
    for with_cycle, topo in ((False, "real"), (True, "real"), (True, "int")):
        m = build_ilp(eg, costs, filt, with_cycle=with_cycle, topo=topo)
        om = O.oracle_build_ilp(oeg, ocosts, ofilt, with_cycle=with_cycle, topo=topo)
        assert m.class_order == om["classes"]
        assert m.var_names == om["var_names"]
        assert m.objective == om["objective"]
        assert (m.lb, m.ub) == (om["lb"], om["ub"])
        assert m.rows == om["rows"]


def test_run_optimize_default_ilp_and_solution_import(tmp_path):
    g = bench_graphs.matmul_chain(3)
    p = tmp_path / "g.graph"
    p.write_text(tensor_lang.emit_graph(g))
    res = run_optimize(RunConfig(graph=str(p), k_max=3))
    assert res.stats["ilp.optimal"] == 1
    eg, filt, _ = explore(tensor_lang.make_single_rooted(g), default_rules(), ExploreLimits(k_max=3))
    costs = egraph_costs(eg, CostModel())
    assert res.result.total_cost <= greedy_extract(eg, costs, filt).total_cost + 1e-9
    # export-only run, then import the optimum back as an external solution
    lp = tmp_path / "m.lp"
    out = run_optimize(RunConfig(graph=str(p), k_max=3, emit_lp=str(lp)))
    assert out.result is None and lp.read_text().startswith("\\ tensorsat extraction model")
    m = build_ilp(eg, costs, filt)
    r1 = solve_ilp(m, eg)
    assert r1.total_cost == pytest.approx(res.result.total_cost, rel=1e-9)
    sol = "\n".join(f"x_{n} = 1" for n in set(r1.selection.values()))
    r2 = parse_solution(m, eg, sol)
    assert r2.selection == r1.selection
