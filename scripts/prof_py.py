"""cProfile of saturate + egraph_costs + greedy_extract (host-side overhead)."""
import cProfile, pstats, sys
sys.path.insert(0, '.')
from paper_2101_01332_b200 import models
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.tensor_lang import build_egraph
g = models.MODELS[sys.argv[1] if len(sys.argv) > 1 else "bert"]()
rules = list(default_rules())
def one():
    eg, _ = build_egraph(g)
    filt, rep = saturate(eg, rules, ExploreLimits(k_multi=1))
    res = greedy_extract(eg, egraph_costs(eg, CostModel()), filt)
for _ in range(3): one()
pr = cProfile.Profile(); pr.enable(); one(); pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(25)
