"""Config-5 congruence cascade: 10M-node e-graph, union w_{2k} ~ w_{2k+1}, rebuild (ncu captures)."""
import ctypes as C
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2101_01332_b200 import _lib, bench_graphs
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.tensor_lang import build_egraph
n = 1415
lib = _lib.load()
g = bench_graphs.matmul_chain(n)
merge = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
eg, classes = build_egraph(g)
saturate(eg, merge, ExploreLimits(n_max=10**9, k_max=1, k_multi=1))
a = np.array([classes[f"w{2 * k}"] for k in range(n // 2)], np.uint32)
b = np.array([classes[f"w{2 * k + 1}"] for k in range(n // 2)], np.uint32)
_lib.check(eg._h, lib.tsat_union_batch(eg._h, len(a), a.ctypes.data_as(C.POINTER(C.c_uint32)), b.ctypes.data_as(C.POINTER(C.c_uint32))))
_lib.check(eg._h, lib.tsat_rebuild(eg._h))
print(eg.num_nodes)
