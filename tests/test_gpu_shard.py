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
