"""Batched e-matching of all 13 canonical patterns on the config-5 10M-node e-graph (ncu captures)."""
import ctypes as C
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2101_01332_b200 import _lib, bench_graphs
from paper_2101_01332_b200.egraph import compile_ruleset
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.tensor_lang import build_egraph
lib = _lib.load()
g = bench_graphs.matmul_chain(1415)
merge = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
eg, classes = build_egraph(g)
saturate(eg, merge, ExploreLimits(n_max=10**9, k_max=1, k_multi=1))
blob, pidx = compile_ruleset(eg, list(default_rules()))
lib.tsat_load_rules(eg._h, len(blob), blob.ctypes.data_as(C.POINTER(C.c_int64)))
pids = np.arange(len(pidx), dtype=np.int32)
counts = np.zeros(len(pidx), np.int64)
for _ in range(3):
    _lib.check(eg._h, lib.tsat_ematch_batch(eg._h, len(pids), pids.ctypes.data_as(C.POINTER(C.c_int32)),
                                            counts.ctypes.data_as(C.POINTER(C.c_int64))))
print(counts.tolist())
