"""Cost-TABLE fixtures made by the REFERENCE (cost.py:135-196, 225-247).

Run in the build container only (needs /root/reference):
    python tests/golden/make_costtable_golden.py
Writes tests/golden/costtable_golden.json.

For each case the reference explores a graph, then a cost table is written in
the reference's text format from the signature keys of the explored e-graph
(signature_key, cost.py:135-140): about half of the keys present (so the rest
fall back to the synthetic formula), with the parameter lists shuffled so
load_cost_table's normalize_signature (cost.py:143-155) has work to do, a few
keys no node has, comments and blank lines.  The fixture stores the table
text, the reference's egraph_costs vector (exact floats), the greedy result
under that vector, and for the strict variant the UnknownSignature message.
"""

from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

from tensorsat import bench as rbench  # noqa: E402
from tensorsat import explorer as rexp  # noqa: E402
from tensorsat import tensor_lang as rtl  # noqa: E402
from tensorsat.cost import egraph_costs, load_cost_table, signature_key  # noqa: E402
from tensorsat.errors import NoFiniteExtraction, UnknownSignature  # noqa: E402
from tensorsat.extract import greedy_extract  # noqa: E402
from tensorsat.rules import default_rules  # noqa: E402
from tensorsat.tensor_lang import SIGNATURES, ValueKind  # noqa: E402

import cases  # noqa: E402

CASES = [
    ("mm3-k2", ["matmul_chain", [3]], 2, 4),
    ("rnn2-k1", ["rnn_cell_stack", [2]], 1, 4),
    ("conv3-k2", ["conv_fanout", [3]], 2, 3),
    ("incep1-k2", ["inception_block", [1]], 2, 3),
    ("gen-mm-k2", ["generate", "matmul-chain", 3, 11], 2, 3),
    ("gen-rnn-k1", ["generate", "rnn-cell-stack", 2, 5], 1, 3),
]


def node_keys(eg):
    """Signature key of every live e-node with children, exactly as
    egraph_costs builds its node_cost arguments (cost.py:225-247)."""
    keys = set()
    for node in eg.iter_nodes():
        if not node.children or node.op in ("input", "weight", "noop"):
            continue
        scalars, shapes = [], []
        for child in node.children:
            v = eg.eclass(child).analysis
            if v.kind == ValueKind.N:
                scalars.append(v.ival)
            elif v.kind == ValueKind.S:
                scalars.append(v.sval)
            elif v.kind == ValueKind.T:
                shapes.append(v.shape)
            else:
                shapes.append(v.pair)
        keys.add(signature_key(node.op, scalars, shapes))
    return sorted(keys)


def shuffle_params(key: str, rng: random.Random) -> str:
    if "[" not in key:
        return key
    head, rest = key.split("[", 1)
    params, tail = rest.split("]", 1)
    ps = params.split(",")
    rng.shuffle(ps)
    return f"{head}[{', '.join(ps)}]{tail}"


def table_text(keys, rng: random.Random):
    lines = ["# cost table written by make_costtable_golden.py", ""]
    chosen = [k for k in keys if rng.random() < 0.5]
    for k in chosen:
        lines.append(f"{shuffle_params(k, rng)} = {rng.uniform(0.001, 2.0)!r}  # measured")
    lines.append("matmul[activation=3](7x7,7x7) = 1.5")
    lines.append("ewadd(3x3,3x3) = 0.25")
    return "\n".join(lines) + "\n", chosen


def main():
    out = []
    for cid, spec, k_multi, k_max in CASES:
        g = cases.build_graph(rbench, rtl, spec)
        eg, filt, _ = rexp.explore(g, list(default_rules()), rexp.ExploreLimits(k_multi=k_multi, k_max=k_max))
        keys = node_keys(eg)
        rng = random.Random(cid)
        text, chosen = table_text(keys, rng)
        model = load_cost_table(text)
        costs = egraph_costs(eg, model)
        rec = {"id": cid, "graph": spec, "k_multi": k_multi, "k_max": k_max, "table": text,
               "n_keys": len(keys), "n_table_hits": len(chosen),
               "costs": {str(k): v for k, v in sorted(costs.items())}}
        try:
            res = greedy_extract(eg, costs, filt)
            rec["greedy"] = {"selection": {str(k): v for k, v in sorted(res.selection.items())},
                             "total": res.total_cost}
        except NoFiniteExtraction:
            rec["greedy"] = {"error": "NoFiniteExtraction"}
        try:
            egraph_costs(eg, load_cost_table(text, strict=True))
            rec["strict_error"] = None
        except UnknownSignature as e:
            rec["strict_error"] = str(e)
        print(cid, len(keys), len(chosen), rec["strict_error"])
        out.append(rec)
    with open(os.path.join(HERE, "costtable_golden.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
