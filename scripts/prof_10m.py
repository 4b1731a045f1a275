"""Per-phase host/device breakdown of the config-5 search (matmul_chain(1415) + merge-shared-lhs)."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from paper_2101_01332_b200 import _lib, bench_graphs
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.tensor_lang import build_egraph

G = ["rebuild", "ematch", "apply_seq", "apply_wave", "reach", "cycles", "costs", "greedy", "snapshot"]
lib = _lib.load()
g = bench_graphs.matmul_chain(1415)
merge = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
for i in range(3):
    t0 = time.perf_counter()
    eg, _ = build_egraph(g)
    t1 = time.perf_counter()
    ms = np.zeros(9); by = np.zeros(9); la = np.zeros(9, np.int64)
    f = lambda r: lib.tsat_kernel_stats(eg._h, ms.ctypes.data_as(C.POINTER(C.c_double)), by.ctypes.data_as(C.POINTER(C.c_double)), la.ctypes.data_as(C.POINTER(C.c_int64)), 9, r)
    f(1)
    t2 = time.perf_counter()
    filt, rep = saturate(eg, merge, ExploreLimits(n_max=10**9, k_max=1, k_multi=1))
    t3 = time.perf_counter()
    ph = np.zeros(32)
    lib.tsat_phase_times(eg._h, ph.ctypes.data_as(C.POINTER(C.c_double)), 32)
    costs = egraph_costs(eg, CostModel()); t4 = time.perf_counter()
    res = greedy_extract(eg, costs, filt); t5 = time.perf_counter()
    f(0)
    print(f"[{i}] build {1e3*(t1-t0):.1f} saturate {1e3*(t3-t2):.1f} costs {1e3*(t4-t3):.1f} greedy {1e3*(t5-t4):.1f} ms")
    print("   phases(ms) snap %.2f reach %.2f ematch %.2f apply %.2f rebuild %.2f cycles %.2f" % tuple(ph[:6]))
    print("   kgroups(ms/launches): " + "  ".join(f"{G[k]} {ms[k]:.2f}/{la[k]}" for k in range(9)))
    del eg, costs, res, filt
