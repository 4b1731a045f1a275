"""World-size-2 gloo tests of the multi-GPU e-matching shard logic.

Each rank e-matches only root e-classes in its id range (shard.class_range)
with the CPU oracle, the ranks' lists are all-gathered over gloo, and the
rank-order concatenation must equal the single-process match list -- the
property the device all-gather (csrc/shard.cu) relies on.  The C-ABI's
tsat_shard_range must use the same partition.
"""

import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import tsat_oracle as O  # noqa: E402
from paper_2101_01332_b200 import bench_graphs, shard  # noqa: E402
from paper_2101_01332_b200.rules import default_rules  # noqa: E402


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_ematch(eg, pattern, filt, lo, hi):
    """Oracle e-matching restricted to root classes in [lo, hi)."""
    found = set()
    for c in sorted(eg.members):
        if not lo <= c < hi:
            continue
        for sub in eg._mc(pattern, c, {}, filt):
            found.add((c, tuple(sorted(sub.items()))))
    return sorted(found, key=lambda m: (m[0], tuple(x for _, x in m[1])))


def _worker(rank, world, port, graph, k_max, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rules = list(default_rules())
        eg, filt, _ = O.oracle_explore(graph, rules, k_multi=1, k_max=k_max)
        pats = []
        for r in rules:
            for cp in r.canonical_sources:
                if cp.pattern not in pats:
                    pats.append(cp.pattern)
        lo, hi = shard.class_range(eg.allocated_nodes, rank, world)
        bad = 0
        total = 0
        for pat in pats:
            full = eg.ematch(pat, frozenset(filt))
            mine = _local_ematch(eg, pat, frozenset(filt), lo, hi)
            assert mine == shard.shard_matches(full, eg.allocated_nodes, rank, world)
            parts = [None] * world
            dist.all_gather_object(parts, mine)
            if shard.concat_rank_matches(parts) != full:
                bad += 1
            total += len(full)
        q.put((rank, bad, total))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("graph,k_max", [("matmul_chain", 2), ("inception_block", 2)])
def test_sharded_ematch_concat_equals_global(graph, k_max):
    g = bench_graphs.matmul_chain(4) if graph == "matmul_chain" else bench_graphs.inception_block(2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, g, k_max, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(q.get(timeout=5) for _ in procs)
    assert all(p.exitcode == 0 for p in procs)
    assert [r[1] for r in res] == [0, 0]
    assert res[0][2] == res[1][2] > 0


def test_class_ranges_partition():
    for n in (0, 1, 7, 100, 10_009_713):
        for w in (1, 2, 3, 4, 8):
            rs = [shard.class_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))


def test_c_abi_shard_range_matches_python():
    from paper_2101_01332_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libtsat.so not built")
    for n in (0, 5, 123457, 10_009_713, (1 << 32) - 5):
        for w in (1, 2, 4, 8):
            for r in range(w):
                assert shard.lib_class_range(n, r, w) == shard.class_range(n, r, w)
