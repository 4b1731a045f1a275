"""Time limit (reference explorer.py:198-201 checks it before every combo):
the device loops read the deadline on the device clock -- before every combo
on the exact path, before every wave in the wave loop -- so one long rule
application cannot overrun the limit by its own length.  A timed-out search
stops with reason "timeout", every counted combo has exactly one outcome, and
the e-graph it leaves is consistent (rebuilt, extractable)."""
import pytest

from paper_2101_01332_b200 import models
from paper_2101_01332_b200.cost import CostModel, egraph_costs
from paper_2101_01332_b200.explorer import ExploreLimits, explore
from paper_2101_01332_b200.extract import greedy_extract
from paper_2101_01332_b200.rules import default_rules

pytestmark = pytest.mark.gpu


def _outcomes(st):
    return (st.skipped_self + st.skipped_compat + st.skipped_shape + st.skipped_cycle + st.applied
            + st.applied_noop)


@pytest.mark.parametrize("limit", [0.0005, 0.002, 0.005])
def test_time_limit_stops_inside_the_apply(limit):
    g = models.MODELS["bert"]()
    rules = list(default_rules())
    explore(g, rules, ExploreLimits(k_multi=1))  # warm the engine pool / caches
    eg, filt, rep = explore(g, rules, ExploreLimits(k_multi=1, time_limit_s=limit))
    assert rep.stop_reason == "timeout"
    # a wave or a rule prologue past the deadline, not a whole iteration (~3 ms) or search (~11 ms)
    assert rep.time_s < limit + 0.004
    for name, st in rep.rules.items():
        assert st.found == _outcomes(st), name
    res = greedy_extract(eg, egraph_costs(eg, CostModel()), filt)
    assert res.total_cost > 0
