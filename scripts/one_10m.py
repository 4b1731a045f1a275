"""One config-5 search (matmul_chain(1415) + merge-shared-lhs, k_max=1) after a warm-up (ncu captures)."""
import sys
sys.path.insert(0, '.')
from paper_2101_01332_b200 import bench_graphs
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.tensor_lang import build_egraph
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1415
g = bench_graphs.matmul_chain(n)
rules = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
for i in range(2):
    eg, _ = build_egraph(g)
    filt, rep = saturate(eg, rules, ExploreLimits(n_max=10**9, k_max=1, k_multi=1))
    res = greedy_extract(eg, egraph_costs(eg, CostModel()), filt)
    print(rep.enodes_per_iter, res.total_cost)
    del eg
