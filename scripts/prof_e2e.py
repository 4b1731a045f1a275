"""cProfile of the e2e public-API path (explore -> egraph_costs -> greedy_extract)."""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
from paper_2101_01332_b200 import models
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, explore
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.extract import greedy_extract
g = models.MODELS["bert"]()
rules = list(default_rules())
lim = ExploreLimits(k_multi=1)
def one():
    eg, filt, rep = explore(g, rules, lim, "efficient")
    res = greedy_extract(eg, egraph_costs(eg, CostModel()), filt)
    return res
for _ in range(3): one()
t0 = time.perf_counter(); one(); print("e2e ms", 1e3 * (time.perf_counter() - t0))
pr = cProfile.Profile(); pr.enable(); one(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
