"""Golden fixtures for the end-to-end optimize path, produced by the REFERENCE.

Run in the build container only (needs /root/reference):
    python tests/golden/make_optimize_golden.py
For each case: the input graph file text (emit_graph of a reference bench
generator or of an authored model graph), the reference's
``run_optimize(RunConfig(..., extractor="greedy"))`` output graph (emit_graph)
and its non-time stats.  Pins cli.run_optimize + greedy_extract + reconstruct
(tests/test_gpu_optimize.py) without the reference being present.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

from tensorsat import bench as rbench  # noqa: E402
from tensorsat import cli as rcli  # noqa: E402
from tensorsat import tensor_lang as rtl  # noqa: E402

CASES = [
    # id, graph source, n_max, k_max, k_multi, filter
    ("matmul_chain4-k2", ("bench", "matmul_chain", 4), 50000, 15, 2, "efficient"),
    ("rnn_cell_stack3-k1", ("bench", "rnn_cell_stack", 3), 50000, 15, 1, "efficient"),
    ("conv_fanout3-k2", ("bench", "conv_fanout", 3), 20000, 15, 2, "efficient"),
    ("inception_block2-k1", ("bench", "inception_block", 2), 20000, 15, 1, "efficient"),
    ("matmul_chain6-k1-none", ("bench", "matmul_chain", 6), 50000, 3, 1, "none"),
    ("nasrnn-k0", ("model", "nasrnn", None), 50000, 15, 0, "efficient"),
    ("bert2-k1", ("model", "bert2", None), 8000, 15, 1, "efficient"),
    ("squeezenet-k2", ("model", "squeezenet", None), 100000, 15, 2, "efficient"),
]


def graph_text(src):
    kind, name, n = src
    if kind == "bench":
        g = getattr(rbench, name)(n)
        return rtl.emit_graph(g)
    # authored model graphs (this repo's models.py) re-emitted through the repo's emitter
    sys.path.insert(0, ROOT)
    from paper_2101_01332_b200 import models, tensor_lang as ltl

    g = models.bert(layers=2) if name == "bert2" else models.MODELS[name]()
    return ltl.emit_graph(g)


def main():
    out = []
    for cid, src, n_max, k_max, k_multi, mode in CASES:
        text = graph_text(src)
        with tempfile.NamedTemporaryFile("w", suffix=".graph", delete=False) as f:
            f.write(text)
            path = f.name
        cfg = rcli.RunConfig(graph=path, n_max=n_max, k_max=k_max, k_multi=k_multi, extractor="greedy",
                             filter_mode=mode)
        res = rcli.run_optimize(cfg)
        os.unlink(path)
        stats = {k: v for k, v in res.stats.items() if "time" not in k}
        out.append({"id": cid, "graph": text, "n_max": n_max, "k_max": k_max, "k_multi": k_multi,
                    "filter_mode": mode, "out_graph": rtl.emit_graph(res.graph), "stats": stats})
        print(cid, stats["cost.before"], stats["cost.after"], stats["graph.nodes_out"])
    json.dump(out, open(os.path.join(HERE, "optimize_golden.json"), "w"), indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
