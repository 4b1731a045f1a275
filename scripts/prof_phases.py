"""Per-phase breakdown of one explore+costs+greedy (phase_ms slots of the engine
+ CUDA-event kernel-group stats).  Usage: python scripts/prof_phases.py [model] [k_multi]"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from paper_2101_01332_b200 import models, _lib
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.tensor_lang import build_egraph

G = ["rebuild", "ematch", "apply_seq", "apply_wave", "reach", "cycles", "costs", "greedy", "snapshot"]
name = sys.argv[1] if len(sys.argv) > 1 else "bert"
km = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nmax = int(sys.argv[3]) if len(sys.argv) > 3 else 50000
lib = _lib.load()
g = models.MODELS[name]()
rules = list(default_rules())
for i in range(int(__import__("os").environ.get("REPS", "4"))):
    eg, _ = build_egraph(g)
    ms = np.zeros(9); by = np.zeros(9); la = np.zeros(9, np.int64)
    f = lambda r: lib.tsat_kernel_stats(eg._h, ms.ctypes.data_as(C.POINTER(C.c_double)), by.ctypes.data_as(C.POINTER(C.c_double)), la.ctypes.data_as(C.POINTER(C.c_int64)), 9, r)
    f(1)
    t0 = time.perf_counter()
    filt, rep = saturate(eg, rules, ExploreLimits(k_multi=km, n_max=nmax))
    t1 = time.perf_counter()
    ph = np.zeros(32)
    lib.tsat_phase_times(eg._h, ph.ctypes.data_as(C.POINTER(C.c_double)), 32)
    dbg = np.zeros(13, np.int64)
    lib.tsat_debug_info(eg._h, dbg.ctypes.data_as(C.POINTER(C.c_int64)), 13)
    costs = egraph_costs(eg, CostModel()); t2 = time.perf_counter()
    res = greedy_extract(eg, costs, filt); t3 = time.perf_counter()
    f(0)
    print(f"[{i}] saturate {1e3*(t1-t0):.1f} costs {1e3*(t2-t1):.1f} greedy {1e3*(t3-t2):.1f} total {1e3*(t3-t0):.1f} ms nodes {rep.enodes_per_iter} iters {rep.iterations}")
    print("   levels %d peeled %d classes %d class-edges %d alloc %d live %d | cudaMallocs so far %d (%.1f MB) engines %d | host syncs %d launches %d" % (dbg[0], dbg[1], dbg[2], dbg[3], dbg[6], dbg[7], dbg[8], dbg[9] / 1e6, dbg[10], dbg[11], dbg[12]))
    print("   phases(ms) snap %.2f reach %.2f ematch %.2f apply %.2f rebuild %.2f cycles %.2f | waves %d hazards %d why %s resolved %d+%d" % (
        ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], ph[8], ph[9], ph[10:16].astype(int).tolist(), ph[28], ph[29]))
    names = ["gates", "accept", "resolve", "candchk", "conflicts", "stops", "boundary", "commit", "unions", "insert", "bookkeep", "top"]
    print("   wave-cta phases(ms): " + " ".join(f"{n} {ph[16+k]:.2f}" for k, n in enumerate(names)))
    print("   kgroups(ms/launches): " + "  ".join(f"{G[k]} {ms[k]:.2f}/{la[k]}" for k in range(9)))
    del eg
