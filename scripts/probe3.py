import sys, time
sys.path.insert(0, '.')
from paper_2101_01332_b200 import models
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.tensor_lang import build_egraph
name = sys.argv[1] if len(sys.argv) > 1 else "bert"
km = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = models.MODELS[name]()
rules = list(default_rules())
for i in range(6):
    t0 = time.perf_counter(); eg, _ = build_egraph(g); t1 = time.perf_counter()
    filt, rep = saturate(eg, rules, ExploreLimits(k_multi=km)); t2 = time.perf_counter()
    costs = egraph_costs(eg, CostModel()); t3 = time.perf_counter()
    res = greedy_extract(eg, costs, filt); t4 = time.perf_counter()
    print(f"{name} build {1e3*(t1-t0):.1f} ms  saturate {1e3*(t2-t1):.1f} ms  costs {1e3*(t3-t2):.1f} ms  greedy {1e3*(t4-t3):.1f} ms  total {1e3*(t4-t0):.1f} ms  nodes {rep.enodes_per_iter[-1]}")
    del eg
