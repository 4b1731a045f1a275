"""Small end-to-end workload for compute-sanitizer (scripts/sanitize.sh):
explore + costs + greedy + ILP skeleton on reference golden cases (wave path,
sequential path, cycles, vanilla mode, levels pre-filter and bitset
pre-filter), each checked against its golden so a sanitizer run is also a
parity run."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]

import cases  # noqa: E402
from paper_2101_01332_b200 import bench_graphs, tensor_lang  # noqa: E402
from paper_2101_01332_b200.cost import CostModel, egraph_costs  # noqa: E402
from paper_2101_01332_b200.explorer import ExploreLimits, saturate  # noqa: E402
from paper_2101_01332_b200.extract import build_ilp, greedy_extract  # noqa: E402
from paper_2101_01332_b200.rules import default_rules  # noqa: E402
from paper_2101_01332_b200.tensor_lang import build_egraph  # noqa: E402

WANT = {"chain3_all_k2", "feedback3_both", "rnn3_all", "incep1_all_k2", "ew_mix", "split_concat",
        "feedback2_lhs_vanilla", "chain4_limit30"}
E = [c for c in json.load(open(os.path.join(ROOT, "tests", "golden", "explore_golden.json"))) if c["id"] in WANT]
n = 0
for budget in (0, 1 << 40):
    for c in E:
        g = cases.build_graph(bench_graphs, tensor_lang, c["graph"])
        rules = cases.select_rules(default_rules(), c["rules"])
        eg, _ = build_egraph(g)
        eg.reach_budget = budget
        filt, rep = saturate(eg, rules, ExploreLimits(**c["limits"]), c["filter_mode"], filt=set(),
                             allow_self_pairs=c["allow_self_pairs"])
        assert eg.dump() == c["final_dump"], c["id"]
        costs = egraph_costs(eg, CostModel())
        if "error" not in c["greedy"]:
            res = greedy_extract(eg, costs, filt)
            assert {str(k): v for k, v in sorted(res.selection.items())} == c["greedy"]["selection"], c["id"]
            build_ilp(eg, costs, filt)
        n += 1
print(f"sanitize driver ok: {n} runs")
