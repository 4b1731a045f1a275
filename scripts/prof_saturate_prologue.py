import sys, time, ctypes as C
sys.path.insert(0,'.')
import torch
from paper_2101_01332_b200 import models, _lib
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.egraph import compile_ruleset
from paper_2101_01332_b200.tensor_lang import build_egraph
g = models.MODELS['bert'](); rules = list(default_rules()); lib=_lib.load()
for i in range(5):
    eg,_ = build_egraph(g); torch.cuda.synchronize()
    t0=time.perf_counter(); eg.set_filter(set()); t1=time.perf_counter()
    blob,_ = compile_ruleset(eg, rules); t2=time.perf_counter()
    _lib.check(eg._h, lib.tsat_load_rules(eg._h, len(blob), _lib.ptr(blob, C.c_int64))); torch.cuda.synchronize(); t3=time.perf_counter()
    print("set_filter %.3f compile %.3f load_rules %.3f ms" % ((t1-t0)*1e3,(t2-t1)*1e3,(t3-t2)*1e3))
    del eg
