"""Efficient pre-filter without the O(C^2) descendants bitset (SURVEY 7(2),
row a10): reaches(leaf, out) (reference cycles.py:52-57, 151-169) answered
from the Kahn peel levels of the snapshot class graph plus a pruned search.
Forced on (reach budget 0), every efficient-mode golden case must still give
the reference's per-iteration dumps, filter lists and stats; with the private
search budget at 0 (TSAT_REACH_STEPS=0, read once per process, so those runs
go through a subprocess) every query the levels cannot decide takes the exact
one-thread path.  The level mode is the default (budget 0); the bitset mode
is kept for budgets that fit it and tested here too."""

import json
import os
import subprocess
import sys

import pytest

import cases
from paper_2101_01332_b200 import bench_graphs, models, tensor_lang
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.tensor_lang import build_egraph, emit_graph, make_single_rooted, parse_graph

import make_model_golden as MG

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(__file__), "golden")
EXPLORE = [c for c in json.load(open(os.path.join(HERE, "explore_golden.json"))) if c["filter_mode"] == "efficient"]
MODELS = json.load(open(os.path.join(HERE, "model_golden.json")))


def _stats(rep):
    return {k: v for k, v in rep.to_stats().items() if "time" not in k}


def run_case_levels(case, budget=0):
    g = cases.build_graph(bench_graphs, tensor_lang, case["graph"])
    rules = cases.select_rules(default_rules(), case["rules"])
    L = case["limits"]
    eg, _ = build_egraph(g)
    eg.reach_budget = budget
    filt = set()
    for i, snap in enumerate(case["iterations"]):
        lim = ExploreLimits(n_max=L["n_max"], k_max=1, k_multi=1 if i < L["k_multi"] else 0)
        filt, rep = saturate(eg, rules, lim, "efficient", filt=filt, allow_self_pairs=case["allow_self_pairs"])
        assert eg.reach_mode == (1 if budget == 0 else 0)
        assert eg.dump() == snap["dump"], f"iteration {i}"
        assert sorted(filt) == snap["filt"], f"iteration {i}"
        if rep.stop_reason != "iter-limit":
            break
    eg2, _ = build_egraph(g)
    eg2.reach_budget = budget
    filt2, rep2 = saturate(eg2, rules, ExploreLimits(**L), "efficient", filt=set(),
                           allow_self_pairs=case["allow_self_pairs"])
    assert eg2.dump() == case["final_dump"]
    assert sorted(filt2) == case["final_filt"]
    assert _stats(rep2) == case["stats"]


@pytest.mark.parametrize("case", EXPLORE, ids=[c["id"] for c in EXPLORE])
def test_levels_prefilter_matches_reference(case):
    run_case_levels(case)


@pytest.mark.parametrize("case", EXPLORE, ids=[c["id"] for c in EXPLORE])
def test_bitset_prefilter_matches_reference(case):
    """The descendants-bitset mode (a budget that fits) on the same cases."""
    run_case_levels(case, budget=1 << 40)


def test_levels_prefilter_exact_path_matches_reference():
    """Same cases with the private search budget at 0 (exact path for every
    query the level filter cannot decide), in a fresh process."""
    code = ("import sys, json; sys.path[:0] = sys.argv[1:3]; import test_gpu_reach_levels as T\n"
            "for c in T.EXPLORE: T.run_case_levels(c)\nprint('ok', len(T.EXPLORE))")
    env = dict(os.environ, TSAT_REACH_STEPS="0")
    tests = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(tests)
    r = subprocess.run([sys.executable, "-c", code, tests, HERE, root], env=env, cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("case", MODELS, ids=[c["id"] for c in MODELS])
def test_levels_prefilter_model_graphs_match_reference(case):
    g = make_single_rooted(parse_graph(emit_graph(models.MODELS[case["model"]]())))
    eg, _ = build_egraph(g)
    eg.reach_budget = 0
    filt, rep = saturate(eg, list(default_rules()),
                         ExploreLimits(n_max=case["n_max"], k_max=case["k_max"], k_multi=case["k_multi"]),
                         "efficient", filt=set())
    assert _stats(rep) == case["stats"]
    assert MG.sha(eg.dump()) == case["final_dump_sha"]
    assert MG.sha(MG.filt_text(filt)) == case["final_filt_sha"]
    res = greedy_extract(eg, egraph_costs(eg, CostModel()), filt)
    assert MG.sha(MG.selection_text(res.selection)) == case["selection_sha"]


def test_second_efficient_iteration_above_a_million_classes():
    """matmul_chain(600) + merge-lhs: iteration 1 leaves 1,800,603 e-nodes in
    1,080,603 classes, whose descendants bitset would need ~146 GB; iteration 2
    runs on the level pre-filter (default budget) up to the node limit."""
    n = 600
    g = bench_graphs.matmul_chain(n)
    rules = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
    eg, _ = build_egraph(g)
    n_max = 2_000_000
    filt, rep = saturate(eg, rules, ExploreLimits(n_max=n_max, k_max=2, k_multi=2), "efficient", filt=set())
    assert rep.iterations == 2
    assert rep.eclasses_per_iter[0] == 3 * n * n + n + 3
    assert rep.enodes_per_iter[0] == 5 * n * n - n + 3
    assert eg.reach_mode == 1
    assert rep.stop_reason == "node-limit"
    assert rep.enodes_per_iter[1] >= n_max
