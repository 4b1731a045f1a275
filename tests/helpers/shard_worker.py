"""One rank of a host-transport shard group (tests/test_gpu_shard_exchange.py).

Launched twice with RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT set; both
ranks use cuda:0.  Each explores the same graph with e-matching split by
e-class range and the match lists all-gathered over torch.distributed (gloo)
through the engine's host transport, then extracts greedily (wide levels
split across the ranks, {cost, node} all-gathered).  Every rank writes its
results; the test compares them with the CPU oracle."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import torch.distributed as dist  # noqa: E402

from paper_2101_01332_b200 import bench_graphs, shard  # noqa: E402
from paper_2101_01332_b200.cost import CostModel, egraph_costs  # noqa: E402
from paper_2101_01332_b200.explorer import ExploreLimits, explore  # noqa: E402
from paper_2101_01332_b200.extract import greedy_extract  # noqa: E402
from paper_2101_01332_b200.rules import default_rules  # noqa: E402

import make_model_golden as MG  # noqa: E402


def main(out_path):
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    exchanged = [0]
    orig = dist.all_gather

    def counting_all_gather(parts, src, group=None):
        exchanged[0] += src.numel()
        return orig(parts, src, group=group)

    dist.all_gather = counting_all_gather
    res = []
    for spec in json.loads(os.environ["SHARD_CASES"]):
        name, args, rule_names, lim = spec
        g = getattr(bench_graphs, name)(*args)
        rules = [r for r in default_rules() if not rule_names or r.name in rule_names]
        before = exchanged[0]
        eg, filt, rep = explore(g, rules, ExploreLimits(**lim), "efficient", shard_group=True)
        after_explore = exchanged[0]
        costs = egraph_costs(eg, CostModel())
        sel = greedy_extract(eg, costs, filt)
        res.append({"case": spec, "dump_sha": MG.sha(eg.dump()), "filt": sorted(filt),
                    "stats": {k: v for k, v in rep.to_stats().items() if "time" not in k},
                    "selection_sha": MG.sha(MG.selection_text(sel.selection)), "total": sel.total_cost,
                    "bytes_explore": after_explore - before, "bytes_greedy": exchanged[0] - after_explore,
                    "shard_range": shard.class_range(eg.allocated_nodes, rank, dist.get_world_size())})
    with open(out_path, "w") as f:
        json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
