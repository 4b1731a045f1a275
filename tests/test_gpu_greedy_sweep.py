"""The reached-selection top-down level sweep (csrc/extract.cu k_sel_cta /
k_sel_wide) against the reference goldens.  The engine picks the sweep only
for graphs with >= 256 single-class levels, so the golden cases run in a
subprocess with TSAT_SEL=2 (sweep forced); plus a 300-deep noop spine that
takes the sweep on its own, against the CPU oracle."""

import json
import os
import subprocess
import sys

import pytest

from oracle import tsat_oracle as O
from paper_2101_01332_b200 import bench_graphs
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.explorer import ExploreLimits, explore
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.rules import default_rules

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, os, sys
sys.path.insert(0, os.path.join(sys.argv[1], "tests", "golden"))
sys.path.insert(0, sys.argv[1])
import cases
from paper_2101_01332_b200 import bench_graphs, tensor_lang
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.errors import NoFiniteExtraction
from paper_2101_01332_b200.explorer import ExploreLimits, explore
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.rules import default_rules
bad = []
for case in json.load(open(os.path.join(sys.argv[1], "tests", "golden", "explore_golden.json"))):
    g = cases.build_graph(bench_graphs, tensor_lang, case["graph"])
    rules = cases.select_rules(default_rules(), case["rules"])
    eg, filt, _ = explore(g, rules, ExploreLimits(**case["limits"]), case["filter_mode"],
                          allow_self_pairs=case["allow_self_pairs"])
    costs = egraph_costs(eg, CostModel())
    if "error" in case["greedy"]:
        try:
            greedy_extract(eg, costs, filt)
            bad.append(case["id"])
        except NoFiniteExtraction:
            pass
        continue
    res = greedy_extract(eg, costs, filt)
    sel = {str(k): v for k, v in sorted(res.selection.items())}
    if sel != case["greedy"]["selection"] or abs(res.total_cost - case["greedy"]["total"]) > 1e-9 * max(1.0, abs(case["greedy"]["total"])):
        bad.append(case["id"])
print(json.dumps(bad))
"""


def test_forced_sweep_matches_reference_goldens():
    env = dict(os.environ, TSAT_SEL="2")
    out = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert json.loads(out.stdout.strip().splitlines()[-1]) == []


def test_deep_spine_sweep_matches_oracle():
    g = bench_graphs.matmul_chain(300)  # noop spine: ~300 single-class levels
    rules = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
    lim = dict(n_max=50000, k_max=0, k_multi=0)
    eg, filt, _ = explore(g, rules, ExploreLimits(**lim))
    oeg, ofilt, _ = O.oracle_explore(g, rules, **lim)
    assert eg.dump() == oeg.dump()
    res = greedy_extract(eg, egraph_costs(eg, CostModel()), filt)
    sel, total, _ = O.oracle_greedy(oeg, O.oracle_costs(oeg, CostModel()), ofilt)
    assert res.selection == sel
    assert res.total_cost == pytest.approx(total, rel=1e-12)
