"""GPU parity: the CUDA engine (through the C-ABI) against reference golden
fixtures and against the CPU oracle on seeded fuzz inputs.

Bar: byte-identical e-graph dump after every iteration, identical filter
lists and non-time stats, identical greedy selection, totals within 1e-9
relative (fp64 sums; the reference sums a Python set, order differs)."""

import json
import os
import random

import pytest

import cases
from oracle import tsat_oracle as O
from paper_2101_01332_b200 import bench_graphs, tensor_lang
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.egraph import EGraph
from paper_2101_01332_b200.errors import NoFiniteExtraction
from paper_2101_01332_b200.explorer import ExploreLimits, explore, saturate
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.rules import default_rules, parse_rules
from paper_2101_01332_b200.sexpr import parse
from paper_2101_01332_b200.tensor_lang import build_egraph

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(__file__), "golden")
EXPLORE = json.load(open(os.path.join(HERE, "explore_golden.json")))
GENERIC = json.load(open(os.path.join(HERE, "generic_golden.json")))


def _stats(rep):
    return {k: v for k, v in rep.to_stats().items() if "time" not in k}


@pytest.mark.parametrize("case", EXPLORE, ids=[c["id"] for c in EXPLORE])
def test_explore_matches_reference_golden(case):
    g = cases.build_graph(bench_graphs, tensor_lang, case["graph"])
    rules = cases.select_rules(default_rules(), case["rules"])
    lim = ExploreLimits(**case["limits"])
    eg, filt, rep = explore(g, rules, lim, case["filter_mode"], allow_self_pairs=case["allow_self_pairs"])
    assert eg.dump() == case["final_dump"]
    assert sorted(filt) == case["final_filt"]
    assert _stats(rep) == case["stats"]
    costs = egraph_costs(eg, CostModel())
    assert {str(k): costs[k] for k in costs} == case["costs"]
    if "error" in case["greedy"]:
        with pytest.raises(NoFiniteExtraction):
            greedy_extract(eg, costs, filt)
    else:
        res = greedy_extract(eg, costs, filt)
        assert {str(k): v for k, v in sorted(res.selection.items())} == case["greedy"]["selection"]
        assert res.total_cost == pytest.approx(case["greedy"]["total"], rel=1e-9)


@pytest.mark.parametrize("case", EXPLORE, ids=[c["id"] for c in EXPLORE])
def test_every_iteration_matches_reference(case):
    """Drive saturate one iteration at a time; dump + filter after each must
    equal the reference's per-iteration snapshot."""
    g = cases.build_graph(bench_graphs, tensor_lang, case["graph"])
    rules = cases.select_rules(default_rules(), case["rules"])
    L = case["limits"]
    eg, _ = build_egraph(g)
    filt = set()
    for i, snap in enumerate(case["iterations"]):
        lim = ExploreLimits(n_max=L["n_max"], k_max=1, k_multi=1 if i < L["k_multi"] else 0)
        filt, rep = saturate(eg, rules, lim, case["filter_mode"], filt=filt,
                             allow_self_pairs=case["allow_self_pairs"])
        assert eg.dump() == snap["dump"], f"iteration {i}"
        assert sorted(filt) == snap["filt"], f"iteration {i}"
        if rep.stop_reason != "iter-limit":
            break


@pytest.mark.parametrize("rec", GENERIC["random"], ids=lambda r: f"seed{r['seed']}")
def test_generic_egraph_ops_and_ematch(rec):
    eg = EGraph()
    ids = []
    for step in cases.random_generic_ops(rec["seed"]):
        if step[0] == "add":
            ids.append(eg.add_enode(step[1], [ids[i] for i in step[2]]))
        elif step[0] == "union":
            eg.union(ids[step[1]], ids[step[2]])
        else:
            eg.rebuild()
    assert ids == rec["ids"]
    assert eg.dump() == rec["dump"]
    for p, want in rec["matches"].items():
        got = [[m.eclass, [list(b) for b in m.bindings]] for m in eg.ematch(parse(p))]
        assert got == want, p


def test_toy_saturation_matches_reference():
    toy = parse_rules(cases.TOY_RULES_TEXT)
    eg = EGraph()
    root = eg.add_term(parse("(div (mul a 2) 2)"))
    eg.root = root
    eg.add_term(parse("a"))
    filt, rep = saturate(eg, toy, ExploreLimits(k_max=10), filter_mode="efficient")
    want = GENERIC["toy"]
    assert eg.dump() == want["dump"]
    assert sorted(filt) == want["filt"]
    assert _stats(rep) == want["stats"]


def _fuzz_specs(n, seed0):
    rng = random.Random(seed0)
    fams = ["matmul-chain", "rnn-cell-stack", "conv-fanout", "inception-block"]
    out = []
    for i in range(n):
        fam = fams[i % 4]
        size = rng.randint(1, 3 if fam != "inception-block" else 2)
        out.append((["generate", fam, size, rng.randint(0, 10**6)], rng.choice([0, 1, 2]), rng.choice([2, 3, 4])))
    return out


@pytest.mark.parametrize("spec", _fuzz_specs(24, 77), ids=lambda s: f"{s[0][1]}-{s[0][2]}-{s[0][3]}")
def test_fuzz_against_oracle(spec):
    gspec, k_multi, k_max = spec
    g = cases.build_graph(bench_graphs, tensor_lang, gspec)
    rules = list(default_rules())
    kw = dict(n_max=3000, k_max=k_max, k_multi=min(k_multi, k_max))
    oeg, ofilt, orep = O.oracle_explore(g, rules, **kw)
    eg, filt, rep = explore(g, rules, ExploreLimits(**kw))
    assert eg.dump() == oeg.dump()
    assert sorted(filt) == sorted(ofilt)
    assert _stats(rep) == {k: v for k, v in orep.to_stats().items() if "time" not in k}
    costs = egraph_costs(eg, CostModel())
    ocosts = O.oracle_costs(oeg, CostModel())
    assert dict(costs) == ocosts
    res = greedy_extract(eg, costs, filt)
    osel, ototal, _ = O.oracle_greedy(oeg, ocosts, ofilt)
    assert res.selection == osel
    assert res.total_cost == pytest.approx(ototal, rel=1e-9)


def test_feedback_cycles_filtered_match_oracle():
    for n in (2, 3, 4, 5):
        g = bench_graphs.matmul_feedback(n)
        rules = [r for r in default_rules() if r.name.startswith("matmul-merge")]
        oeg, ofilt, orep = O.oracle_explore(g, rules, k_multi=2, k_max=3, n_max=5000)
        eg, filt, rep = explore(g, rules, ExploreLimits(k_multi=2, k_max=3, n_max=5000))
        assert eg.dump() == oeg.dump()
        assert sorted(filt) == sorted(ofilt)
        assert _stats(rep) == {k: v for k, v in orep.to_stats().items() if "time" not in k}


_FILTERED = [c for c in EXPLORE if c["filter_mode"] != "none"]


@pytest.mark.parametrize("case", _FILTERED, ids=[c["id"] for c in _FILTERED])
def test_on_reject_matches_reference(case):
    """on_reject (post-iteration variant) sees the reference's rejected combos
    in the reference's order; recording (efficient: exact sequential path)
    leaves the result unchanged."""
    g = cases.build_graph(bench_graphs, tensor_lang, case["graph"])
    rules = cases.select_rules(default_rules(), case["rules"])
    got = []

    def on_reject(_eg, _filt, rule, matches):
        got.append([rule.name, [[m.eclass, [list(b) for b in m.bindings]] for m in matches]])

    eg, filt, rep = explore(g, rules, ExploreLimits(**case["limits"]), case["filter_mode"],
                            on_reject=on_reject, allow_self_pairs=case["allow_self_pairs"])
    assert got == case["rejects"]
    assert eg.dump() == case["final_dump"]
    assert sorted(filt) == case["final_filt"]
    assert _stats(rep) == case["stats"]


def test_vanilla_against_oracle_and_slower_than_efficient():
    """C5 shape (pkg/tests/test_acceptance.py:240-253): one k_multi iteration of
    matmul-merge-shared-lhs on matmul_chain(33) in both modes; each equals the
    oracle, and the efficient pre-filter beats per-combo apply-and-check."""
    g = bench_graphs.matmul_chain(33)
    rules = cases.select_rules(default_rules(), cases.MERGE_LHS)
    lim = ExploreLimits(k_multi=1, k_max=1)
    out = {}
    for mode in ("efficient", "vanilla"):
        eg, filt, rep = explore(g, rules, lim, mode)
        oeg, ofilt, orep = O.oracle_explore(g, rules, filter_mode=mode, n_max=lim.n_max, k_max=1, k_multi=1)
        assert eg.dump() == oeg.dump(), mode
        assert sorted(filt) == sorted(ofilt), mode
        assert _stats(rep) == {k: v for k, v in orep.to_stats().items() if "time" not in k}, mode
        out[mode] = rep
    assert out["efficient"].rules["matmul-merge-shared-lhs"].found >= 1000
    assert out["efficient"].time_s < out["vanilla"].time_s


@pytest.mark.parametrize("case", EXPLORE[::3], ids=[c["id"] for c in EXPLORE[::3]])
def test_tsat_iterate_matches_reference_per_iteration(case):
    """The per-iteration C entry point (tsat_iterate through explorer.iterate):
    iteration i of the caller's loop gates the multi-pattern rules itself."""
    from paper_2101_01332_b200.explorer import iterate

    g = cases.build_graph(bench_graphs, tensor_lang, case["graph"])
    rules = cases.select_rules(default_rules(), case["rules"])
    lim = ExploreLimits(**case["limits"])
    eg, _ = build_egraph(g)
    filt = set()
    for i, snap in enumerate(case["iterations"]):
        filt, rep = iterate(eg, rules, i, lim, case["filter_mode"], filt=filt,
                            allow_self_pairs=case["allow_self_pairs"])
        assert eg.dump() == snap["dump"], f"iteration {i}"
        assert sorted(filt) == snap["filt"], f"iteration {i}"
        if rep.stop_reason != "iter-limit":
            break
