"""Per-iteration fixtures for the authored model graphs, made by the REFERENCE.

Run in the build container only (needs /root/reference):
    python tests/golden/make_model_golden.py            # the six model graphs
    python tests/golden/make_model_golden.py config5    # configs[4] (~10 min, ~20 GB RSS)

The graphs are this package's authored models (paper_2101_01332_b200/models.py)
written out in the reference's `tensorgraph v1` text format and parsed back by
the REFERENCE parser (tensor_lang.py:640-700), so everything downstream of the
text -- build_egraph, every iteration of saturate, egraph_costs, greedy_extract
-- is the reference's own code.  After every iteration (explorer.py:264-267,
wrapped like make_golden.py does) the fixture stores the sha256 of dump() and
of the sorted filter list plus the node/class counts; at the end the non-time
stats, the sha256 of the cost vector (repr of every float, id order), the
sha256 of the greedy selection and the greedy total.  Hashes keep the fixture
small (BERT's final dump is ~5 MB); the GPU test recomputes the same hashes.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)


def sha(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()


def filt_text(filt) -> str:
    return ",".join(str(i) for i in sorted(filt))


def costs_text(costs) -> str:
    return "\n".join(f"{k}:{costs[k]!r}" for k in sorted(costs))


def selection_text(sel) -> str:
    return "\n".join(f"{k}:{sel[k]}" for k in sorted(sel))


# (id, model, k_multi, n_max, k_max) -- the bench configurations (bench.py WORKLOADS)
MODEL_CASES = [
    ("nasrnn-k0-n50000", "nasrnn", 0, 50000, 15),
    ("bert-k1-n50000", "bert", 1, 50000, 15),
    ("squeezenet-k2-n100000", "squeezenet", 2, 100000, 15),
    ("resnext50-k2-n100000", "resnext50", 2, 100000, 15),
    ("inception_v3-k2-n50000", "inception_v3", 2, 50000, 15),
    ("nasnet_a-k2-n50000", "nasnet_a", 2, 50000, 15),
]


def graph_text(model: str) -> str:
    from paper_2101_01332_b200 import models
    from paper_2101_01332_b200.tensor_lang import emit_graph

    return emit_graph(models.MODELS[model]())


def run_reference(text: str, rule_names, k_multi, n_max, k_max):
    sys.path.insert(0, "/root/reference/pkg/src")
    from tensorsat import explorer as rexp
    from tensorsat.cost import CostModel, egraph_costs
    from tensorsat.extract import greedy_extract
    from tensorsat.rules import default_rules
    from tensorsat.tensor_lang import make_single_rooted, parse_graph

    g = make_single_rooted(parse_graph(text))  # emit_graph drops the noop plumbing (tensor_lang.py:685-688)
    rules = [r for r in default_rules() if rule_names is None or r.name in rule_names]
    iters = []
    orig_end = rexp._Engine.end_iteration

    def end_iteration(self):
        orig_end(self)
        iters.append({"dump_sha": sha(self.eg.dump()), "filt_sha": sha(filt_text(self.filt)),
                      "nodes": self.eg.num_nodes, "classes": self.eg.num_classes})

    rexp._Engine.end_iteration = end_iteration
    t0 = time.perf_counter()
    try:
        eg, filt, rep = rexp.explore(g, rules, rexp.ExploreLimits(n_max=n_max, k_max=k_max, k_multi=k_multi),
                                     "efficient")
    finally:
        rexp._Engine.end_iteration = orig_end
    t_explore = time.perf_counter() - t0
    costs = egraph_costs(eg, CostModel())
    res = greedy_extract(eg, costs, filt)
    t_all = time.perf_counter() - t0
    stats = {k: v for k, v in rep.to_stats().items() if "time" not in k}
    return {"iterations": iters, "stats": stats, "final_dump_sha": sha(eg.dump()),
            "final_filt_sha": sha(filt_text(filt)), "costs_sha": sha(costs_text(costs)),
            "selection_sha": sha(selection_text(res.selection)), "selection_size": len(res.selection),
            "total": res.total_cost, "ref_seconds": {"explore": t_explore, "explore_costs_greedy": t_all}}


def main_models():
    out = []
    for cid, model, k_multi, n_max, k_max in MODEL_CASES:
        text = graph_text(model)
        rec = {"id": cid, "model": model, "k_multi": k_multi, "n_max": n_max, "k_max": k_max,
               "graph_sha": sha(text)}
        rec.update(run_reference(text, None, k_multi, n_max, k_max))
        print(cid, len(rec["iterations"]), rec["stats"].get("stop_reason"), rec["ref_seconds"], flush=True)
        out.append(rec)
    with open(os.path.join(HERE, "model_golden.json"), "w") as f:
        json.dump(out, f, indent=1)


def main_config5(n: int = 1415):
    """configs[4]: matmul_chain(n) + [matmul-merge-shared-lhs], k_multi=1, k_max=1."""
    from paper_2101_01332_b200 import bench_graphs
    from paper_2101_01332_b200.tensor_lang import emit_graph

    text = emit_graph(bench_graphs.matmul_chain(n))
    rec = {"id": f"config5-matmul_chain{n}", "n": n, "rules": ["matmul-merge-shared-lhs"], "k_multi": 1,
           "n_max": 10 ** 9, "k_max": 1, "graph_sha": sha(text)}
    rec.update(run_reference(text, {"matmul-merge-shared-lhs"}, 1, 10 ** 9, 1))
    print(rec["id"], rec["iterations"], rec["stats"], rec["ref_seconds"], flush=True)
    with open(os.path.join(HERE, f"config5_golden_n{n}.json"), "w") as f:
        json.dump(rec, f, indent=1)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "config5":
        main_config5(int(sys.argv[2]) if len(sys.argv) > 2 else 1415)
    else:
        main_models()
