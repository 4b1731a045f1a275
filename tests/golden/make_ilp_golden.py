"""Generate ILP golden fixtures by running the REFERENCE implementation.

Run in the build container only (needs /root/reference):
    python tests/golden/make_ilp_golden.py
For a few explored e-graphs of cases.EXPLORE_CASES: reachable classes, the
exported LP text (no cycle constraints / real / int topological order) and
the reference solver's optimum.  Pins csrc/ilp.cu + extract.build_ilp /
export_lp / solve_ilp (tests/test_gpu_ilp.py).
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
from tensorsat import extract as rext  # noqa: E402
from tensorsat import tensor_lang as rtl  # noqa: E402
from tensorsat.cost import CostModel, egraph_costs  # noqa: E402
from tensorsat.rules import default_rules  # noqa: E402

import cases  # noqa: E402

ILP_CASES = ["chain2_lhs", "feedback3_both", "feedback2_lhs_none", "rnn2_all", "commute", "mm_assoc",
             "conv_relu", "incep1_all_k2", "ew_mix"]
VARIANTS = [("none", False, "real"), ("real", True, "real"), ("int", True, "int")]


def main():
    by_id = {c[0]: c for c in cases.EXPLORE_CASES}
    out = []
    for cid in ILP_CASES:
        _, gspec, names, limits, mode, self_pairs = by_id[cid]
        g = cases.build_graph(rbench, rtl, gspec)
        rules = cases.select_rules(default_rules(), names)
        eg, filt, _ = rexp.explore(g, rules, rexp.ExploreLimits(**limits), mode,
                                   allow_self_pairs=self_pairs)
        costs = egraph_costs(eg, CostModel())
        rec = {"id": cid, "reachable": rext.reachable_classes(eg, set(filt), eg.root), "variants": []}
        for vname, with_cycle, topo in VARIANTS:
            m = rext.build_ilp(eg, costs, filt, with_cycle=with_cycle, topo=topo)
            v = {"variant": vname, "with_cycle": with_cycle, "topo": topo, "lp": rext.export_lp(m),
                 "num_vars": m.num_vars, "num_rows": len(m.rows)}
            try:
                r = rext.solve_ilp(m, eg, 60.0)
                v["total"] = r.total_cost
                v["selection"] = {str(k): val for k, val in sorted(r.selection.items())}
                v["optimal"] = r.optimal
            except Exception as e:  # noqa: BLE001 - record the reference's failure class
                v["error"] = type(e).__name__
            rec["variants"].append(v)
        out.append(rec)
        print(cid, [(v["variant"], v.get("total", v.get("error")), v["num_rows"]) for v in rec["variants"]])
    with open(os.path.join(HERE, "ilp_golden.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
