"""Forced full congruence round on the config-5 10M-node e-graph (ncu captures)."""
import sys
sys.path.insert(0, '.')
from paper_2101_01332_b200 import _lib, bench_graphs
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.tensor_lang import build_egraph
lib = _lib.load()
g = bench_graphs.matmul_chain(1415)
merge = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
eg, _ = build_egraph(g)
saturate(eg, merge, ExploreLimits(n_max=10**9, k_max=1, k_multi=1))
for _ in range(3):
    _lib.check(eg._h, lib.tsat_force_rebuild(eg._h))
print(eg.num_nodes)
