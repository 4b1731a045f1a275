import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_01332_b200 import bench_graphs
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.tensor_lang import build_egraph
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1415
merge = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
eg, _ = build_egraph(bench_graphs.matmul_chain(n))
filt, rep = saturate(eg, merge, ExploreLimits(n_max=10**9, k_max=1, k_multi=1))
res = greedy_extract(eg, egraph_costs(eg, CostModel()), filt)
print(rep.enodes_per_iter, res.total_cost)
