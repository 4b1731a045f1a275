"""Host-side split of one e2e step (explore -> egraph_costs -> greedy_extract through
the public API): wall time of each host stage around the device work."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_01332_b200 import models  # noqa: E402
from paper_2101_01332_b200.cost import CostModel, egraph_costs  # noqa: E402
from paper_2101_01332_b200.explorer import ExploreLimits, saturate  # noqa: E402
from paper_2101_01332_b200.extract import greedy_extract  # noqa: E402
from paper_2101_01332_b200.rules import default_rules  # noqa: E402
from paper_2101_01332_b200.tensor_lang import build_egraph, initial_enodes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bert"
if name == "bert":
    g = models.MODELS["bert"]()
    rules = list(default_rules())
    lim = ExploreLimits(k_multi=1)
else:  # a bench.py workload (e.g. synth10m)
    import bench
    g, rules, w = bench.build_workload(name)
    lim = ExploreLimits(n_max=w["n_max"], k_max=w["k_max"], k_multi=w["k_multi"])
for rep in range(6):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    initial_enodes(g)
    t.append(time.perf_counter())
    eg, _ = build_egraph(g)
    t.append(time.perf_counter())
    filt, r = saturate(eg, rules, lim, "efficient")
    t.append(time.perf_counter())
    costs = egraph_costs(eg, CostModel())
    t.append(time.perf_counter())
    res = greedy_extract(eg, costs, filt)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    if name != "bert" and rep == 5:
        import cProfile
        import pstats
        eg2, _ = build_egraph(g)
        pr = cProfile.Profile()
        pr.enable()
        f2, _ = saturate(eg2, rules, lim, "efficient")
        c2 = egraph_costs(eg2, CostModel())
        greedy_extract(eg2, c2, f2)
        torch.cuda.synchronize()
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(15)
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print("initial_enodes %.3f build_egraph(incl.) %.3f saturate %.3f costs %.3f greedy %.3f | total %.3f ms" %
          (d[0], d[1], d[2], d[3], d[4], sum(d[1:])))
    del eg
