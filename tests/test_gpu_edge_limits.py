"""Edge cases of the iteration control (reference explorer.py:311-365,
198-206): no iterations, an empty rule set, a node limit below the initial
e-graph (the budget check precedes found++, so nothing is counted), a node
limit hit inside the first rule, a one-node graph, and k_multi above k_max --
each against the CPU oracle (dump, filter list, every non-time statistic)."""
import pytest

from oracle import tsat_oracle as O
from paper_2101_01332_b200 import bench_graphs, models
from paper_2101_01332_b200.explorer import ExploreLimits, explore
from paper_2101_01332_b200.rules import default_rules
from paper_2101_01332_b200.tensor_lang import TensorGraph, make_identifier, make_single_rooted

pytestmark = pytest.mark.gpu


def _stats(rep):
    return {k: v for k, v in rep.to_stats().items() if "time" not in k}


def one_node():
    g = TensorGraph()
    g.add("x", "input", identifier=make_identifier("x", (8, 8)))
    g.set_outputs(["x"])
    return make_single_rooted(g)


CASES = [
    ("k_max0", lambda: bench_graphs.matmul_chain(3), "all", dict(k_max=0, k_multi=0, n_max=5000)),
    ("no_rules", lambda: bench_graphs.matmul_chain(3), "none", dict(k_max=5, k_multi=1, n_max=5000)),
    ("n_max_below_initial", lambda: bench_graphs.matmul_chain(4), "all", dict(k_max=5, k_multi=1, n_max=3)),
    ("n_max_inside_first_rule", lambda: models.MODELS["nasrnn"](), "all", dict(k_max=5, k_multi=0, n_max=383)),
    ("n_max_inside_first_iteration", lambda: models.MODELS["nasrnn"](), "all", dict(k_max=5, k_multi=0, n_max=418)),
    ("one_node", one_node, "all", dict(k_max=5, k_multi=2, n_max=5000)),
    ("k_multi_eq_k_max", lambda: bench_graphs.matmul_feedback(4), "all", dict(k_max=2, k_multi=2, n_max=5000)),
]


@pytest.mark.parametrize("name,graph,rules,lim", CASES, ids=[c[0] for c in CASES])
def test_iteration_control_edges_match_oracle(name, graph, rules, lim):
    g = graph()
    rs = [] if rules == "none" else list(default_rules())
    eg, filt, rep = explore(g, rs, ExploreLimits(**lim))
    oeg, ofilt, orep = O.oracle_explore(g, rs, **lim)
    assert rep.stop_reason == orep.stop_reason
    assert eg.dump() == oeg.dump()
    assert sorted(filt) == sorted(ofilt)
    assert _stats(rep) == {k: v for k, v in orep.to_stats().items() if "time" not in k}


def test_bad_limits_raise_like_the_reference():
    # ExploreLimits validation (reference explorer.py:63-67)
    with pytest.raises(ValueError):
        ExploreLimits(k_max=2, k_multi=5)
    with pytest.raises(ValueError):
        ExploreLimits(n_max=-1)
