import sys, time
sys.path.insert(0, '.')
import ctypes as C, numpy as np
from paper_2101_01332_b200 import models, _lib
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, explore, saturate
from paper_2101_01332_b200.tensor_lang import build_egraph
lib = _lib.load()
rules = list(default_rules())
name = sys.argv[1] if len(sys.argv) > 1 else "bert"
km = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = models.MODELS[name]()
eg, _ = build_egraph(g)
filt = set()
for it in range(15):
    t = time.time()
    filt, rep = saturate(eg, rules, ExploreLimits(k_max=1, k_multi=1 if it < km else 0, n_max=50000), filt=filt)
    ph = np.zeros(16)
    lib.tsat_phase_times(eg._h, ph.ctypes.data_as(C.POINTER(C.c_double)), 16)
    print(it, rep.stop_reason, rep.enodes_per_iter, "%.3fs" % (time.time() - t), "phases", np.round(ph[:6], 1), "waves", ph[8], "hazards", ph[9], "why", ph[10:16])
    for nm, s in rep.rules.items():
        if s.found: print("   ", nm, s)
    if rep.stop_reason != "iter-limit": break
info = np.zeros(8, np.int64)
lib.tsat_debug_info(eg._h, info.ctypes.data_as(C.POINTER(C.c_int64)), 8)
print("levels", info[0], "trimmed", info[1], "classes", info[2], "edges", info[3])
