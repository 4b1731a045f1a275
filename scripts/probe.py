import sys, time
sys.path.insert(0, '.')
import ctypes as C, numpy as np
from paper_2101_01332_b200 import models, _lib
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, explore
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.extract import greedy_extract
lib = _lib.load()
for name, kw in [("bert", dict(k_multi=1)), ("nasrnn", dict(k_multi=0)), ("squeezenet", dict(k_multi=2, n_max=100000))]:
    g = models.MODELS[name]()
    for rep_i in range(2):
        t = time.time()
        eg, filt, rep = explore(g, list(default_rules()), ExploreLimits(**kw))
        t1 = time.time() - t
        ph = np.zeros(8)
        lib.tsat_phase_times(eg._h, ph.ctypes.data_as(C.POINTER(C.c_double)), 8)
        costs = egraph_costs(eg, CostModel())
        res = greedy_extract(eg, costs, filt)
        print(name, rep.stop_reason, rep.enodes_per_iter, "explore %.3fs total %.3fs" % (t1, time.time() - t), res.total_cost, "phases(ms)", np.round(ph, 1))
