"""Shared case corpus for golden fixtures and parity tests.

A case spec is plain data so both the reference (in this container, via
make_golden.py) and the B200 engine / oracle (anywhere) rebuild the same
input graph and rule list from it.
"""

from __future__ import annotations

import random

MERGE_LHS = ["matmul-merge-shared-lhs"]
MERGE_BOTH = ["matmul-merge-shared-lhs", "matmul-merge-shared-rhs"]

TOY_RULES_TEXT = """
mul2-to-shift: (mul ?x 2) => (shl ?x 1)
mul-div-assoc: (div (mul ?x ?y) ?z) => (mul ?x (div ?y ?z))
div-self-to-one: (div ?x ?x) => 1
mul-one: (mul ?x 1) => ?x
"""


def build_graph(mod_bench, mod_tl, spec):
    """spec: [family, args...]; mod_bench / mod_tl are the generator and
    tensor_lang modules of whichever implementation builds the graph."""
    kind = spec[0]
    if kind == "generate":
        _, name, size, seed = spec
        return mod_bench.generate(name, size, None if seed is None else random.Random(seed))
    if kind == "custom":
        return _custom(mod_tl, spec[1])
    fn = getattr(mod_bench, kind)
    return fn(*spec[1], **(spec[2] if len(spec) > 2 else {}))


def _custom(tl, name):
    g = tl.TensorGraph()
    if name == "commute":
        g.add("a", "input", identifier="a@4_4")
        g.add("b", "input", identifier="b@4_4")
        g.add("s", "ewadd", ("a", "b"))
        g.set_outputs(["s"])
    elif name == "transpose2":
        g.add("x", "input", identifier="x@3_5")
        g.add("t1", "transpose", ("x",), perm="1_0")
        g.add("t2", "transpose", ("t1",), perm="1_0")
        g.set_outputs(["t2"])
    elif name == "conv_relu":
        g.add("x", "input", identifier="x@1_8_9_9")
        g.add("w", "weight", identifier="w@16_8_3_3")
        g.add("c", "conv", ("x", "w"), stride_h=1, stride_w=1, padding=0, activation=0)
        g.add("r", "relu", ("c",))
        g.set_outputs(["r"])
    elif name == "ew_mix":
        # associativity + commutativity chains: exercises stale-hashcons
        # duplicates
        for v in "abcd":
            g.add(v, "input", identifier=f"{v}@8_8")
        g.add("s1", "ewadd", ("a", "b"))
        g.add("s2", "ewadd", ("s1", "c"))
        g.add("s3", "ewadd", ("s2", "d"))
        g.add("p1", "ewmul", ("a", "c"))
        g.add("p2", "ewmul", ("p1", "s1"))
        g.set_outputs(["s3", "p2"])
    elif name == "mm_assoc":
        g.add("a", "input", identifier="a@8_16")
        g.add("b", "weight", identifier="b@16_32")
        g.add("c", "weight", identifier="c@32_8")
        g.add("d", "weight", identifier="d@8_4")
        g.add("m1", "matmul", ("a", "b"), activation=0)
        g.add("m2", "matmul", ("m1", "c"), activation=0)
        g.add("m3", "matmul", ("m2", "d"), activation=0)
        g.add("r", "relu", ("m3",))
        g.set_outputs(["r"])
    elif name == "split_concat":
        g.add("a", "input", identifier="a@4_6")
        g.add("b", "input", identifier="b@4_6")
        g.add("c", "concat_2", ("a", "b"), axis=1)
        g.add("s", "split", ("c",), axis=1)
        g.add("l", "split_0", ("s",))
        g.add("r", "split_1", ("s",))
        g.add("e", "ewadd", ("l", "r"))
        g.set_outputs(["e"])
    elif name == "inception_concat":
        g.add("x", "input", identifier="x@1_8_9_9")
        for i, k in enumerate((1, 3, 3)):
            g.add(f"w{i}", "weight", identifier=f"w{i}@8_8_{k}_{k}")
            g.add(f"c{i}", "conv", ("x", f"w{i}"), stride_h=1, stride_w=1, padding=0, activation=0)
        g.add("cat", "concat_3", ("c0", "c1", "c2"), axis=1)
        g.add("r", "relu", ("cat",))
        g.set_outputs(["r"])
    else:
        raise KeyError(name)
    return tl.make_single_rooted(g)


def select_rules(all_rules, names):
    if names == "all":
        return list(all_rules)
    return [r for r in all_rules if r.name in names]


def _L(**kw):
    base = {"n_max": 50000, "k_max": 15, "k_multi": 1}
    base.update(kw)
    return base


# (case id, graph spec, rule names, limits, filter_mode, allow_self_pairs)
EXPLORE_CASES = [
    ("chain2_lhs", ["matmul_chain", [2]], MERGE_LHS, _L(), "efficient", False),
    ("chain2_lhs_self", ["matmul_chain", [2]], MERGE_LHS, _L(), "efficient", True),
    ("chain3_lhs_k2", ["matmul_chain", [3]], MERGE_LHS, _L(k_multi=2, k_max=2), "efficient", False),
    ("chain3_all_k2", ["matmul_chain", [3]], "all", _L(k_multi=2, k_max=3), "efficient", False),
    ("chain4_limit30", ["matmul_chain", [4]], MERGE_LHS, _L(n_max=30, k_multi=3, k_max=5), "efficient", False),
    ("chain5_limit200", ["matmul_chain", [5]], "all", _L(n_max=200, k_multi=2, k_max=4), "efficient", False),
    ("feedback2_lhs", ["matmul_feedback", [2]], MERGE_LHS, _L(), "efficient", False),
    ("feedback2_lhs_none", ["matmul_feedback", [2]], MERGE_LHS, _L(), "none", False),
    ("feedback3_both", ["matmul_feedback", [3]], MERGE_BOTH, _L(k_max=2), "efficient", False),
    ("feedback4_all", ["matmul_feedback", [4]], "all", _L(k_max=3), "efficient", False),
    ("rnn2_all", ["rnn_cell_stack", [2]], "all", _L(), "efficient", False),
    ("rnn3_all_k0", ["rnn_cell_stack", [3]], "all", _L(k_multi=0), "efficient", False),
    ("rnn3_all", ["rnn_cell_stack", [3]], "all", _L(), "efficient", False),
    ("conv2_all", ["conv_fanout", [2]], "all", _L(), "efficient", False),
    ("conv3_all_k2", ["conv_fanout", [3]], "all", _L(k_multi=2), "efficient", False),
    ("incep1_all_k2", ["inception_block", [1]], "all", _L(k_multi=2), "efficient", False),
    ("incep2_all", ["inception_block", [2]], "all", _L(), "efficient", False),
    ("commute", ["custom", "commute"], "all", _L(), "efficient", False),
    ("transpose2", ["custom", "transpose2"], "all", _L(), "efficient", False),
    ("conv_relu", ["custom", "conv_relu"], "all", _L(), "efficient", False),
    ("ew_mix", ["custom", "ew_mix"], "all", _L(k_multi=0), "efficient", False),
    ("ew_mix_none", ["custom", "ew_mix"], "all", _L(k_multi=0, k_max=6), "none", False),
    ("mm_assoc", ["custom", "mm_assoc"], "all", _L(k_multi=1), "efficient", False),
    ("split_concat", ["custom", "split_concat"], "all", _L(), "efficient", False),
    ("incep_concat", ["custom", "inception_concat"], "all", _L(k_multi=1, k_max=4), "efficient", False),
    ("rand_mm_1", ["generate", "matmul-chain", 3, 1], MERGE_BOTH, _L(k_max=2), "efficient", False),
    ("rand_rnn_2", ["generate", "rnn-cell-stack", 2, 2], "all", _L(k_max=3), "efficient", False),
    ("rand_conv_3", ["generate", "conv-fanout", 2, 3], "all", _L(k_max=3), "efficient", False),
    ("rand_incep_4", ["generate", "inception-block", 1, 4], "all", _L(k_max=3), "efficient", False),
    ("k0_none", ["matmul_chain", [2]], MERGE_LHS, _L(k_max=0, k_multi=0), "efficient", False),
    ("empty_rules", ["matmul_chain", [2]], [], _L(), "efficient", False),
    # vanilla (apply-on-clone) cycle filtering, cycles.py:248-254
    ("chain3_lhs_vanilla", ["matmul_chain", [3]], MERGE_LHS, _L(k_max=2), "vanilla", False),
    ("feedback2_lhs_vanilla", ["matmul_feedback", [2]], MERGE_LHS, _L(), "vanilla", False),
    ("feedback3_both_vanilla", ["matmul_feedback", [3]], MERGE_BOTH, _L(k_max=2), "vanilla", False),
    ("rnn2_all_vanilla", ["rnn_cell_stack", [2]], "all", _L(k_max=3), "vanilla", False),
    ("ew_mix_vanilla", ["custom", "ew_mix"], "all", _L(k_multi=0, k_max=4), "vanilla", False),
    ("chain4_limit60_vanilla", ["matmul_chain", [4]], MERGE_LHS, _L(n_max=60, k_multi=3, k_max=5), "vanilla", False),
]


def random_generic_ops(seed, n_extra=10, n_unions=3):
    """Operation script for a generic (analysis-free) e-graph, mirroring the
    reference test helper random_egraph (pkg/tests/test_egraph.py:254-266):
    a list of ("add", op, [child op-indices]) / ("union", i, j) / ("rebuild",)."""
    rng = random.Random(seed)
    script = [("add", a, []) for a in ["a", "b", "c", 0]]
    n = 4
    for _ in range(n_extra):
        op = rng.choice(["f", "g", "h", "k"])
        arity = 1 if op in ("f", "g") else 2
        script.append(("add", op, [rng.randrange(n) for _ in range(arity)]))
        n += 1
    for _ in range(n_unions):
        script.append(("union", rng.randrange(n), rng.randrange(n)))
    script.append(("rebuild",))
    return script


GENERIC_PATTERNS = ["(f ?x)", "(h ?x ?y)", "(h ?x ?x)", "(f (g ?x))", "(h (f ?x) ?y)", "(k a ?y)"]
