"""The next iteration's e-matching runs speculatively next to the cycle
check's level peel and is kept only when the check filters
nothing.  Here the check does filter: the fig-3 merge of the reference's
test_cycles.py is applied by hand, closing a loop, so iteration 1's
post-processing (break_all_cycles, reference cycles.py:234-245) filter-lists
a node and iteration 2 must e-match against the new filter list.  The device
run (overlap on, the default) must equal the CPU oracle's, iteration by
iteration, and the run with the overlap disabled."""
import os
import subprocess
import sys

import pytest

from oracle import tsat_oracle as O
from paper_2101_01332_b200.explorer import ExploreLimits, saturate
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.sexpr import parse
from paper_2101_01332_b200.tensor_lang import TensorGraph, build_egraph, make_identifier, make_single_rooted

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def feedback_graph():
    g = TensorGraph()
    g.add("x", "input", identifier=make_identifier("x", (64, 64)))
    g.add("w", "weight", identifier=make_identifier("w", (64, 64)))
    g.add("m2", "matmul", ("x", "w"), activation=0)
    g.add("m3", "matmul", ("x", "m2"), activation=0)
    # element-wise tail: the associativity / commutativity rules keep later
    # iterations changing, so the search reaches iteration 2
    g.add("a1", "ewadd", ("m3", "x"))
    g.add("a2", "ewadd", ("a1", "w"))
    g.add("a3", "ewmul", ("a2", "x"))
    g.set_outputs(["a3"])
    return make_single_rooted(g)


def fig3_merge(eg, classes):
    env = {"act": eg.add_enode(0), "x": classes["x"], "a": classes["w"], "b": classes["m2"]}
    t0 = eg.add_term(parse("(split_0 (split 1 (matmul ?act ?x (concat_2 1 ?a ?b))))"), env)
    t1 = eg.add_term(parse("(split_1 (split 1 (matmul ?act ?x (concat_2 1 ?a ?b))))"), env)
    eg.union(classes["m2"], t0)
    eg.union(classes["m3"], t1)
    eg.rebuild()


LIM = dict(k_multi=2, k_max=4, n_max=5000)


def run_device():
    g = feedback_graph()
    eg, classes = build_egraph(g)
    fig3_merge(eg, classes)
    dumps = []
    filt = set()
    rules = list(default_rules())
    for i in range(LIM["k_max"]):
        filt, rep = saturate(eg, rules, ExploreLimits(**LIM), "efficient", filt, _iteration=i)
        dumps.append((eg.dump(), sorted(filt), rep.postprocess_filtered))
        if rep.stop_reason != "iter-limit":
            break
    eg2, classes2 = build_egraph(g)
    fig3_merge(eg2, classes2)
    filt2, rep2 = saturate(eg2, rules, ExploreLimits(**LIM), "efficient")
    return dumps, eg2.dump(), sorted(filt2), rep2


def test_speculative_ematch_discarded_when_the_cycle_check_filters():
    dumps, final_dump, final_filt, rep = run_device()
    # oracle, same construction
    g = feedback_graph()
    oeg, ocls = O.oracle_build_egraph(g)
    fig3_merge(oeg, ocls)
    want = []

    def snap(eg, filt, r):
        want.append((eg.dump(), sorted(filt)))

    ofilt, orep = O.oracle_saturate(oeg, list(default_rules()), filter_mode="efficient", on_iteration=snap, **LIM)
    assert orep.postprocess_filtered >= 1 and orep.iterations >= 2  # the scenario this test is about
    assert rep.postprocess_filtered == orep.postprocess_filtered
    assert final_dump == oeg.dump()
    assert final_filt == sorted(ofilt)
    assert [(d, f) for d, f, _ in dumps] == want[: len(dumps)]


def test_same_result_with_the_overlap_disabled():
    code = ("import json,sys; sys.path[:0]=[%r, %r]; import test_gpu_overlap_invalidation as T; "
            "d, fd, ff, r = T.run_device(); print(json.dumps([fd, ff, r.postprocess_filtered]))"
            % (ROOT, os.path.join(ROOT, "tests")))
    outs = []
    for env_extra in ({}, {"TSAT_NO_OVERLAP": "1"}):
        env = dict(os.environ, **env_extra)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                   check=True).stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1]
