"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (needs /root/reference):
    python tests/golden/make_golden.py
Writes tests/golden/explore_golden.json and tests/golden/generic_golden.json.
The fixtures pin the CPU oracle (tests/test_oracle_golden.py) and the GPU
engine (tests/test_gpu_parity.py) without the reference being present.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

from tensorsat import bench as rbench  # noqa: E402
from tensorsat import explorer as rexp  # noqa: E402
from tensorsat import tensor_lang as rtl  # noqa: E402
from tensorsat.cost import CostModel, egraph_costs  # noqa: E402
from tensorsat.egraph import EGraph  # noqa: E402
from tensorsat.errors import NoFiniteExtraction  # noqa: E402
from tensorsat.extract import greedy_extract  # noqa: E402
from tensorsat.rules import default_rules, parse_rules  # noqa: E402
from tensorsat.sexpr import parse  # noqa: E402

import cases  # noqa: E402


def run_explore_case(case):
    cid, gspec, names, limits, mode, self_pairs = case
    g = cases.build_graph(rbench, rtl, gspec)
    rules = cases.select_rules(default_rules(), names)
    snaps = []
    orig_end = rexp._Engine.end_iteration

    def end_iteration(self):
        orig_end(self)
        snaps.append({"dump": self.eg.dump(), "filt": sorted(self.filt)})

    rejects = []

    def on_reject(_eg, _filt, rule, matches):
        rejects.append([rule.name, [[m.eclass, [list(b) for b in m.bindings]] for m in matches]])

    rexp._Engine.end_iteration = end_iteration
    try:
        eg, filt, rep = rexp.explore(
            g, rules, rexp.ExploreLimits(**limits), mode, allow_self_pairs=self_pairs,
            on_reject=on_reject,
        )
    finally:
        rexp._Engine.end_iteration = orig_end
    stats = {k: v for k, v in rep.to_stats().items() if "time" not in k}
    out = {"id": cid, "graph": gspec, "rules": names, "limits": limits,
           "filter_mode": mode, "allow_self_pairs": self_pairs,
           "iterations": snaps, "stats": stats, "final_dump": eg.dump(),
           "final_filt": sorted(filt), "rejects": rejects}
    costs = egraph_costs(eg, CostModel())
    out["costs"] = {str(k): v for k, v in sorted(costs.items())}
    try:
        res = greedy_extract(eg, costs, filt)
        out["greedy"] = {"selection": {str(k): v for k, v in sorted(res.selection.items())},
                         "total": res.total_cost}
    except NoFiniteExtraction:
        out["greedy"] = {"error": "NoFiniteExtraction"}
    return out


def run_generic(seed):
    script = cases.random_generic_ops(seed)
    eg = EGraph()
    ids = []
    for step in script:
        if step[0] == "add":
            ids.append(eg.add_enode(step[1], [ids[i] for i in step[2]]))
        elif step[0] == "union":
            eg.union(ids[step[1]], ids[step[2]])
        else:
            eg.rebuild()
    matches = {}
    for p in cases.GENERIC_PATTERNS:
        matches[p] = [[m.eclass, [list(b) for b in m.bindings]] for m in eg.ematch(parse(p))]
    return {"seed": seed, "ids": ids, "dump": eg.dump(), "matches": matches}


def run_toy():
    toy = parse_rules(cases.TOY_RULES_TEXT)
    eg = EGraph()
    root = eg.add_term(parse("(div (mul a 2) 2)"))
    eg.root = root
    eg.add_term(parse("a"))
    filt, rep = rexp.saturate(eg, toy, rexp.ExploreLimits(k_max=10), filter_mode="efficient")
    stats = {k: v for k, v in rep.to_stats().items() if "time" not in k}
    return {"dump": eg.dump(), "filt": sorted(filt), "stats": stats}


def main():
    explore = [run_explore_case(c) for c in cases.EXPLORE_CASES]
    with open(os.path.join(HERE, "explore_golden.json"), "w") as f:
        json.dump(explore, f, indent=0, sort_keys=True)
    generic = {"random": [run_generic(s) for s in range(10)], "toy": run_toy()}
    with open(os.path.join(HERE, "generic_golden.json"), "w") as f:
        json.dump(generic, f, indent=0, sort_keys=True)
    for c in explore:
        print(c["id"], c["stats"]["explore.stop_reason"], c["stats"]["explore.enodes_per_iter"],
              len(c["final_dump"]))


if __name__ == "__main__":
    main()
