"""Launch list of one bench step (configs[1] BERT: saturate + costs + greedy on a
device-resident e-graph) for ncu --profile-from-start off: warm-up steps run
outside the profiler window, the last step inside it."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_01332_b200 import models  # noqa: E402
from paper_2101_01332_b200.cost import CostModel, egraph_costs  # noqa: E402
from paper_2101_01332_b200.explorer import ExploreLimits, saturate  # noqa: E402
from paper_2101_01332_b200.extract import greedy_extract  # noqa: E402
from paper_2101_01332_b200.rules import default_rules  # noqa: E402
from paper_2101_01332_b200.tensor_lang import build_egraph  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bert"
km = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = models.MODELS[name]()
rules = list(default_rules())
for i in range(4):
    eg = build_egraph(g)[0]
    torch.cuda.synchronize()
    if i == 3:
        torch.cuda.profiler.start()
    filt, rep = saturate(eg, rules, ExploreLimits(k_multi=km))
    res = greedy_extract(eg, egraph_costs(eg, CostModel()), filt)
    torch.cuda.synchronize()
    if i == 3:
        torch.cuda.profiler.stop()
    print(rep.enodes_per_iter, res.total_cost)
    del eg
