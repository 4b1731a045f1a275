"""The multi-GPU data plane executed with a real exchange: two
ranks (processes) on the one GPU of the test box, torch.distributed/gloo
moving the bytes through the engine's host transport (tsat_shard_setup_host)
instead of NCCL.  The device code under test is the same as with NCCL: per-
pattern match counts all-gathered, this rank's lists packed, one all-gather,
rank-order unpack into every MatchSet (csrc/shard.cu shard_gather_matches),
and greedy's wide levels split by class slot with the {cost, node} records
all-gathered (csrc/extract.cu).  Both ranks must produce the CPU oracle's
e-graph, filter list, stats and greedy selection."""

import json
import os
import socket
import subprocess
import sys

import pytest

from oracle import tsat_oracle as O
from paper_2101_01332_b200 import bench_graphs
from paper_2101_01332_b200.cost import CostModel
from paper_2101_01332_b200.rules import default_rules

import make_model_golden as MG

pytestmark = pytest.mark.gpu

CASES = [
    ["matmul_chain", [3], [], {"k_multi": 2, "k_max": 4}],
    ["rnn_cell_stack", [3], [], {"k_multi": 1, "k_max": 4}],
    ["inception_block", [2], [], {"k_multi": 2, "k_max": 3, "n_max": 20000}],
    # wide greedy levels (> 8,192 classes): the sharded fold + record all-gather
    ["matmul_chain", [100], ["matmul-merge-shared-lhs"], {"k_multi": 1, "k_max": 1}],
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def rank_results(tmp_path_factory):
    d = tmp_path_factory.mktemp("shard")
    worker = os.path.join(os.path.dirname(__file__), "helpers", "shard_worker.py")
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), SHARD_CASES=json.dumps(CASES))
        procs.append(subprocess.Popen([sys.executable, worker, str(d / f"r{r}.json")], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=900)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-4000:]
    return [json.load(open(d / f"r{r}.json")) for r in range(2)]


@pytest.mark.parametrize("k", range(len(CASES)), ids=[f"{c[0]}{c[1]}" for c in CASES])
def test_two_rank_exchange_matches_oracle(rank_results, k):
    name, args, rule_names, lim = CASES[k]
    g = getattr(bench_graphs, name)(*args)
    rules = [r for r in default_rules() if not rule_names or r.name in rule_names]
    oeg, ofilt, orep = O.oracle_explore(g, rules, **lim)
    ocosts = O.oracle_costs(oeg, CostModel())
    osel, ototal, _ = O.oracle_greedy(oeg, ocosts, ofilt)
    ostats = {k2: v for k2, v in orep.to_stats().items() if "time" not in k2}
    ranges = []
    for r in range(2):
        res = rank_results[r][k]
        assert res["dump_sha"] == MG.sha(oeg.dump()), f"rank {r}"
        assert res["filt"] == sorted(ofilt)
        assert res["stats"] == ostats
        assert res["selection_sha"] == MG.sha(MG.selection_text(osel))
        assert res["total"] == pytest.approx(ototal, rel=1e-9)
        assert res["bytes_explore"] > 0, "no match list crossed the transport"
        ranges.append(res["shard_range"])
    assert ranges[0][1] == ranges[1][0] and ranges[0][0] == 0
    if name == "matmul_chain" and args == [100]:
        assert rank_results[0][k]["bytes_greedy"] > 0, "greedy's wide levels were not exchanged"
