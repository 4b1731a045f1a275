"""End-to-end drop-in path on the GPU: cli.run_optimize (parse -> explore ->
egraph_costs -> greedy_extract -> reconstruct -> emit_graph) against the
reference's own run_optimize outputs (tests/golden/optimize_golden.json,
made by tests/golden/make_optimize_golden.py from /root/reference).
Output graph text must be identical; non-time stats identical (costs within
1e-9 relative: fp64 sums in a different order)."""

import json
import os

import pytest

from paper_2101_01332_b200.cli import RunConfig, run_optimize
from paper_2101_01332_b200.tensor_lang import emit_graph

pytestmark = pytest.mark.gpu

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "optimize_golden.json")))


@pytest.mark.parametrize("case", CASES, ids=[c["id"] for c in CASES])
def test_run_optimize_matches_reference(case, tmp_path):
    p = tmp_path / "in.graph"
    p.write_text(case["graph"])
    res = run_optimize(RunConfig(graph=str(p), n_max=case["n_max"], k_max=case["k_max"], k_multi=case["k_multi"],
                                 extractor="greedy", filter_mode=case["filter_mode"]))
    assert emit_graph(res.graph) == case["out_graph"]
    stats = {k: v for k, v in res.stats.items() if "time" not in k}
    assert set(stats) == set(case["stats"])
    for k, v in case["stats"].items():
        if k.startswith("cost."):
            assert stats[k] == pytest.approx(v, rel=1e-9, abs=1e-12), k
        else:
            assert stats[k] == v, k
