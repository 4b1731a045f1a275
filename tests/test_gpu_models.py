"""GPU parity on the authored benchmark graphs (BASELINE configs 0-3): the
device exploration + extraction must equal the CPU oracle byte for byte
(final dump, filter list, non-time stats, greedy selection; totals within
1e-9 relative, fp64 sums in a different order)."""

import pytest

from oracle import tsat_oracle as O
from paper_2101_01332_b200 import models
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.explorer import ExploreLimits, explore
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.rules import default_rules

pytestmark = pytest.mark.gpu

CASES = [
    ("nasrnn", 0, 50000),        # configs[0]: single-pattern rules only
    ("bert", 1, 6000),           # configs[1] at a reduced node limit (oracle time)
    ("bert", 1, 20000),
    ("bert", 1, 50000),          # configs[1] as benchmarked (soft-writer resolution in every wave)
    ("squeezenet", 2, 100000),   # configs[2]
    ("resnext50", 2, 100000),
    ("inception_v3", 2, 6000),   # configs[3]
    ("inception_v3", 2, 15000),
    ("inception_v3", 2, 50000),
    ("nasnet_a", 2, 50000),
]


def _stats(rep):
    return {k: v for k, v in rep.to_stats().items() if "time" not in k}


@pytest.mark.parametrize("name,k_multi,n_max", CASES, ids=[f"{c[0]}-k{c[1]}-n{c[2]}" for c in CASES])
def test_model_graph_matches_oracle(name, k_multi, n_max):
    g = models.MODELS[name]()
    rules = list(default_rules())
    eg, filt, rep = explore(g, rules, ExploreLimits(k_multi=k_multi, n_max=n_max, k_max=15))
    oeg, ofilt, orep = O.oracle_explore(g, rules, k_multi=k_multi, n_max=n_max, k_max=15)
    assert eg.dump() == oeg.dump()
    assert sorted(filt) == sorted(ofilt)
    assert _stats(rep) == {k: v for k, v in orep.to_stats().items() if "time" not in k}
    costs = egraph_costs(eg, CostModel())
    ocosts = O.oracle_costs(oeg, CostModel())
    assert {int(k): costs[k] for k in costs} == ocosts
    res = greedy_extract(eg, costs, filt)
    osel, ototal, _ = O.oracle_greedy(oeg, ocosts, ofilt)
    assert res.selection == osel
    assert res.total_cost == pytest.approx(ototal, rel=1e-9)
