"""Config 5: matmul_chain(n) + matmul-merge-shared-lhs, k_multi=1, k_max=1."""
import sys, time
sys.path.insert(0, '.')
import ctypes as C, numpy as np
from paper_2101_01332_b200 import bench_graphs, _lib
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.tensor_lang import build_egraph
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1415
lib = _lib.load()
rules = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
g = bench_graphs.matmul_chain(n)
for rep_i in range(2):
    t0 = time.perf_counter(); eg, _ = build_egraph(g); t1 = time.perf_counter()
    filt, rep = saturate(eg, rules, ExploreLimits(n_max=10**9, k_max=1, k_multi=1)); t2 = time.perf_counter()
    costs = egraph_costs(eg, CostModel()); t3 = time.perf_counter()
    res = greedy_extract(eg, costs, filt); t4 = time.perf_counter()
    ms = np.zeros(9); by = np.zeros(9); la = np.zeros(9, np.int64)
    lib.tsat_kernel_stats(eg._h, ms.ctypes.data_as(C.POINTER(C.c_double)), by.ctypes.data_as(C.POINTER(C.c_double)), la.ctypes.data_as(C.POINTER(C.c_int64)), 9, 1)
    print(f"n={n} nodes={rep.enodes_per_iter} classes={rep.eclasses_per_iter} expected N={5*n*n-n+3} C={3*n*n+n+3}")
    print(f"build {t1-t0:.3f}s saturate {t2-t1:.3f}s costs {t3-t2:.3f}s greedy {t4-t3:.3f}s cost={res.total_cost}")
    for name, m, b, l in zip(["rebuild","ematch","apply_seq","apply_wave","reach","cycles","costs","greedy","snapshot"], ms, by, la):
        print(f"   {name:10s} {m:9.2f} ms  {b/1e9:8.3f} GB  {l:6d} launches  {(b/1e9)/(m/1e3) if m else 0:8.1f} GB/s")
    del eg
