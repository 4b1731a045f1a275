"""One BERT explore+costs+greedy after one warm-up (for ncu captures)."""
import sys
sys.path.insert(0, '.')
from paper_2101_01332_b200 import models
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.tensor_lang import build_egraph
name = sys.argv[1] if len(sys.argv) > 1 else "bert"
g = models.MODELS[name]()
rules = list(default_rules())
for i in range(2):
    eg, _ = build_egraph(g)
    filt, rep = saturate(eg, rules, ExploreLimits(k_multi=1))
    res = greedy_extract(eg, egraph_costs(eg, CostModel()), filt)
    print(rep.enodes_per_iter, res.total_cost)
    del eg
