"""on_reject on the wave path: a registered hook no longer routes efficient
mode through the single-thread exact path; the wave engine logs every
cycle-rejected position (device log + exact-path hazards, merged in position
order), and the callbacks see the same combos, in the same order, as the CPU
oracle (reference explorer.py:222-224), with the same final e-graph."""
import pytest

from oracle import tsat_oracle as O
from paper_2101_01332_b200 import bench_graphs, models
from paper_2101_01332_b200.explorer import ExploreLimits, explore
from paper_2101_01332_b200.rules import default_rules

pytestmark = pytest.mark.gpu

# matmul_feedback graphs are built to make the pre-filter reject (the model
# graphs reject nothing at these limits)
CASES = [
    ("feedback6-merge", 6, True, dict(k_multi=2, k_max=3, n_max=5000)),
    ("feedback40-merge", 40, True, dict(k_multi=2, k_max=3, n_max=50000)),
    ("feedback40-all", 40, False, dict(k_multi=2, k_max=4, n_max=50000)),
    ("bert6k", None, False, dict(k_multi=1, k_max=15, n_max=6000)),
]


def _graph(n):
    return models.MODELS["bert"]() if n is None else bench_graphs.matmul_feedback(n)


def _rules(merge_only):
    rules = list(default_rules())
    return [r for r in rules if r.name.startswith("matmul-merge")] if merge_only else rules


@pytest.mark.parametrize("name,n,merge_only,lim", CASES, ids=[c[0] for c in CASES])
def test_on_reject_wave_path_matches_oracle(name, n, merge_only, lim):
    g, rules = _graph(n), _rules(merge_only)
    got = []

    def on_reject(_eg, _filt, rule, matches):
        got.append((rule.name, [(m.eclass, tuple(sorted(m.bindings))) for m in matches]))

    eg, filt, rep = explore(g, rules, ExploreLimits(**lim), "efficient", on_reject=on_reject)
    want = []

    def o_reject(rule, combo):
        want.append((rule.name, [(c, tuple(sorted(s.items()))) for c, s in combo]))

    oeg, ofilt, orep = O.oracle_explore(g, rules, on_reject=o_reject, **lim)
    assert got == want
    assert eg.dump() == oeg.dump()
    assert sorted(filt) == sorted(ofilt)
