"""Device-side e-matching shards on one GPU: each rank's local
part (tsat_shard_setup without an NCCL id = no exchange) is computed on the
same e-graph, and the rank-order concatenation must equal the unsharded
device e-matching and the CPU oracle's."""

import pytest

from oracle import tsat_oracle as O
from paper_2101_01332_b200 import bench_graphs, models, shard
from paper_2101_01332_b200.explorer import ExploreLimits, explore
from paper_2101_01332_b200.rules import default_rules

pytestmark = pytest.mark.gpu


def _patterns(rules):
    pats = []
    for r in rules:
        for cp in r.canonical_sources:
            if cp.pattern not in pats:
                pats.append(cp.pattern)
    return pats


@pytest.mark.parametrize("name", ["matmul_chain", "nasrnn"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_shards_concat_to_global(name, world):
    g = bench_graphs.matmul_chain(6) if name == "matmul_chain" else models.nasrnn(steps=2)
    rules = list(default_rules())
    eg, filt, _ = explore(g, rules, ExploreLimits(k_multi=1, k_max=3))
    oeg, ofilt, _ = O.oracle_explore(g, rules, k_multi=1, k_max=3)
    assert eg.dump() == oeg.dump()
    for pat in _patterns(rules):
        full = eg.ematch(pat, filt)
        parts = []
        for r in range(world):
            shard.attach(eg, r, world)
            parts.append(eg.ematch(pat, filt))
        shard.attach(eg, 0, 1)
        assert shard.concat_rank_matches(parts) == full
        lo_hi = [shard.class_range(eg.allocated_nodes, r, world) for r in range(world)]
        for (lo, hi), part in zip(lo_hi, parts):
            assert all(lo <= m.eclass < hi for m in part)
        om = oeg.ematch(pat, frozenset(ofilt))
        assert [(m.eclass, tuple(x for _, x in m.bindings)) for m in full] == \
               [(c, tuple(x for _, x in b)) for c, b in om]


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_greedy_wide_levels_match(world):
    """Greedy's wide levels split by class slot across W ranks (emulated on one
    GPU without an NCCL id: every slice computed, packed and unpacked) must
    give the unsharded selection and total."""
    from paper_2101_01332_b200.cost import CostModel, egraph_costs
    from paper_2101_01332_b200.extract import greedy_extract

    g = bench_graphs.matmul_chain(150)  # 112k e-nodes, 67k classes: HBM path with wide levels
    merge = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
    eg, filt, rep = explore(g, merge, ExploreLimits(n_max=10**9, k_max=1, k_multi=1))
    costs = egraph_costs(eg, CostModel())
    ref = greedy_extract(eg, costs, filt)
    shard.attach(eg, world - 1, world)
    res = greedy_extract(eg, costs, filt)
    shard.attach(eg, 0, 1)
    assert res.selection == ref.selection
    assert res.total_cost == ref.total_cost
