"""Time greedy_extract / costs / cycle check repeatedly on the final BERT e-graph."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2101_01332_b200 import models
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.tensor_lang import build_egraph
name = sys.argv[1] if len(sys.argv) > 1 else "bert"
g = models.MODELS[name]()
eg, _ = build_egraph(g)
filt, rep = saturate(eg, list(default_rules()), ExploreLimits(k_multi=1))
costs = egraph_costs(eg, CostModel())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cold in (False, True):
    ts = []
    for i in range(10):
        if cold:
            flush.zero_(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = greedy_extract(eg, costs, filt)
        ts.append(time.perf_counter() - t0)
    print(f"greedy {'cold' if cold else 'warm'}: min {1e3*min(ts):.3f} ms median {1e3*sorted(ts)[5]:.3f} ms cost {res.total_cost}")
