"""C5 / Table 7 shape (reference pkg/tests/test_acceptance.py:240-253): one
k_multi iteration of matmul-merge-shared-lhs on matmul_chain(n) with the
efficient pre-filter vs vanilla apply-and-check, on the GPU engine and on the
CPU oracle.  Prints one JSON line per n."""

import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden"))

import cases  # noqa: E402
from oracle import tsat_oracle as O  # noqa: E402
from paper_2101_01332_b200 import bench_graphs  # noqa: E402
from paper_2101_01332_b200.explorer import ExploreLimits, explore  # noqa: E402
from paper_2101_01332_b200.rules import default_rules  # noqa: E402

rules = cases.select_rules(default_rules(), cases.MERGE_LHS)
for n in (int(x) for x in (sys.argv[1:] or ["33"])):
    g = bench_graphs.matmul_chain(n)
    out = {"graph": f"matmul_chain({n})"}
    for mode in ("efficient", "vanilla"):
        explore(g, rules, ExploreLimits(k_multi=1, k_max=1), mode)  # warm
        t = time.perf_counter()
        eg, filt, rep = explore(g, rules, ExploreLimits(k_multi=1, k_max=1), mode)
        out[f"gpu_{mode}_s"] = time.perf_counter() - t
        out["found"] = rep.rules["matmul-merge-shared-lhs"].found
        t = time.perf_counter()
        oeg, ofilt, orep = O.oracle_explore(g, rules, filter_mode=mode, k_max=1, k_multi=1)
        out[f"cpu_{mode}_s"] = time.perf_counter() - t
        out[f"{mode}_identical"] = eg.dump() == oeg.dump() and sorted(filt) == sorted(ofilt)
    out["gpu_ratio_eff_over_van"] = out["gpu_efficient_s"] / out["gpu_vanilla_s"]
    out["cpu_ratio_eff_over_van"] = out["cpu_efficient_s"] / out["cpu_vanilla_s"]
    print(json.dumps(out), flush=True)
