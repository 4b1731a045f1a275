"""Greedy extraction on the config-5 10M-node e-graph, bracketed by
cudaProfilerStart/Stop for ncu --profile-from-start off; prints level stats."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2101_01332_b200 import bench_graphs  # noqa: E402
from paper_2101_01332_b200.cost import CostModel, egraph_costs  # noqa: E402
from paper_2101_01332_b200.explorer import ExploreLimits, saturate  # noqa: E402
from paper_2101_01332_b200.extract import greedy_extract  # noqa: E402
from paper_2101_01332_b200.rules import default_rules  # noqa: E402
from paper_2101_01332_b200.tensor_lang import build_egraph  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1415
merge = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
eg, _ = build_egraph(bench_graphs.matmul_chain(n))
filt, rep = saturate(eg, merge, ExploreLimits(n_max=10**9, k_max=1, k_multi=1))
costs = egraph_costs(eg, CostModel())
for i in range(3):
    torch.cuda.synchronize()
    if i == 2:
        torch.cuda.profiler.start()
    t = time.perf_counter()
    res = greedy_extract(eg, costs, filt)
    dt = time.perf_counter() - t
    if i == 2:
        torch.cuda.profiler.stop()
    print(f"greedy {1e3 * dt:.3f} ms cost {res.total_cost}", flush=True)
