"""Host-side profile of build_egraph (cProfile + wall time) on the GPU box."""
import sys, time, cProfile, pstats
sys.path.insert(0,'.')
import torch
from paper_2101_01332_b200 import models
from paper_2101_01332_b200.tensor_lang import build_egraph
g = models.MODELS['bert']()
for i in range(5):
    eg,_ = build_egraph(g); torch.cuda.synchronize(); del eg
t=time.perf_counter()
for i in range(20):
    eg,_ = build_egraph(g); torch.cuda.synchronize(); del eg
print('build_egraph ms', (time.perf_counter()-t)/20*1e3)
pr=cProfile.Profile(); pr.enable()
for i in range(20):
    eg,_ = build_egraph(g); torch.cuda.synchronize(); del eg
pr.disable(); pstats.Stats(pr).sort_stats('tottime').print_stats(14)
