"""Build the config-5 10M-node e-graph, then run e-matching of all 13 canonical
patterns once (for ncu captures of k_ematch at scale)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_01332_b200 import _lib, bench_graphs
from paper_2101_01332_b200.egraph import compile_ruleset
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.tensor_lang import build_egraph
lib = _lib.load()
merge = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
eg, _ = build_egraph(bench_graphs.matmul_chain(int(sys.argv[1]) if len(sys.argv) > 1 else 1415))
saturate(eg, merge, ExploreLimits(n_max=10**9, k_max=1, k_multi=1))
blob, pidx = compile_ruleset(eg, list(default_rules()))
lib.tsat_load_rules(eg._h, len(blob), blob.ctypes.data_as(C.POINTER(C.c_int64)))
n = C.c_int64(); nb = C.c_int32(); tot = 0
for p in range(len(pidx)):
    lib.tsat_ematch(eg._h, p, None, None, 0, C.byref(n), C.byref(nb)); tot += n.value
print("matches", tot)
