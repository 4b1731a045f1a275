"""Config 5 sweep: on the 10M-node e-graph of matmul_chain(1415) after
one k_multi=1 iteration of matmul-merge-shared-lhs, time (i) e-matching of all 13
canonical patterns, (ii) a forced full rebuild and a congruence-cascade rebuild
after unioning weight classes w_{2k} ~ w_{2k+1}, (iii) costs + greedy.  Prints
per-kernel-group device time, algorithmic bytes and achieved GB/s (JSON)."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_01332_b200 import _lib, bench_graphs  # noqa: E402
from paper_2101_01332_b200.cost import CostModel, egraph_costs  # noqa: E402
from paper_2101_01332_b200.egraph import compile_ruleset  # noqa: E402
from paper_2101_01332_b200.explorer import ExploreLimits, saturate  # noqa: E402
from paper_2101_01332_b200.extract import greedy_extract  # noqa: E402
from paper_2101_01332_b200.rules import default_rules  # noqa: E402
from paper_2101_01332_b200.tensor_lang import build_egraph  # noqa: E402

PROF = os.environ.get("TSAT_PROF_REGION", "")  # ncu --profile-from-start off: capture one region


class region:
    """cudaProfilerStart/Stop around one named region on the last repetition
    (TSAT_PROF_REGION=ematch|rebuild_forced|rebuild_cascade|costs|greedy|search)."""
    last = False

    def __init__(self, name):
        self.on = PROF == name and region.last

    def __enter__(self):
        if self.on:
            import torch
            torch.cuda.synchronize()
            torch.cuda.profiler.start()

    def __exit__(self, *a):
        if self.on:
            import torch
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()


GROUPS = ["rebuild", "ematch", "apply_seq", "apply_wave", "reach", "cycles", "costs", "greedy", "snapshot"]


def kstats(lib, eg, reset=True):
    ms = np.zeros(9); by = np.zeros(9); la = np.zeros(9, np.int64)
    lib.tsat_kernel_stats(eg._h, ms.ctypes.data_as(C.POINTER(C.c_double)), by.ctypes.data_as(C.POINTER(C.c_double)),
                          la.ctypes.data_as(C.POINTER(C.c_int64)), 9, 1 if reset else 0)
    return {g: {"ms": float(m), "bytes": float(b), "launches": int(l)} for g, m, b, l in zip(GROUPS, ms, by, la)}


def run(n=1415, reps=3):
    lib = _lib.load()
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
    merge = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
    g = bench_graphs.matmul_chain(n)
    out = {"n": n}
    best = {}
    for rep in range(reps):
        region.last = rep == reps - 1
        eg, classes = build_egraph(g)
        t0 = time.perf_counter()
        with region("search"):
            filt, report = saturate(eg, merge, ExploreLimits(n_max=10**9, k_max=1, k_multi=1))
        with region("costs"):
            costs = egraph_costs(eg, CostModel())
        with region("greedy"):
            res = greedy_extract(eg, costs, filt)
        t1 = time.perf_counter()
        step = kstats(lib, eg)
        out["nodes"] = report.enodes_per_iter[-1]
        out["classes"] = report.eclasses_per_iter[-1]
        out.setdefault("search_s", []).append(t1 - t0)
        # (i) e-matching of all 13 canonical patterns on the 10M-node e-graph
        blob, pidx = compile_ruleset(eg, list(default_rules()))
        lib.tsat_load_rules(eg._h, len(blob), blob.ctypes.data_as(C.POINTER(C.c_int64)))
        kstats(lib, eg)
        pids = np.arange(len(pidx), dtype=np.int32)
        counts = np.zeros(len(pidx), np.int64)
        with region("ematch"):
            _lib.check(eg._h, lib.tsat_ematch_batch(eg._h, len(pids), pids.ctypes.data_as(C.POINTER(C.c_int32)),
                                                    counts.ctypes.data_as(C.POINTER(C.c_int64))))
        matched = int(counts.sum())
        em = kstats(lib, eg)["ematch"]
        # (ii) forced full rebuild, then a congruence cascade: w_{2k} ~ w_{2k+1}
        with region("rebuild_forced"):
            _lib.check(eg._h, lib.tsat_force_rebuild(eg._h))
        rb = kstats(lib, eg)["rebuild"]
        a = np.array([classes[f"w{2 * k}"] for k in range(n // 2)], np.uint32)
        b = np.array([classes[f"w{2 * k + 1}"] for k in range(n // 2)], np.uint32)
        _lib.check(eg._h, lib.tsat_union_batch(eg._h, len(a), a.ctypes.data_as(C.POINTER(C.c_uint32)),
                                               b.ctypes.data_as(C.POINTER(C.c_uint32))))
        kstats(lib, eg)
        with region("rebuild_cascade"):
            _lib.check(eg._h, lib.tsat_rebuild(eg._h))
        cas = kstats(lib, eg)["rebuild"]
        nodes_after = eg.num_nodes
        cur = {"ematch_13": em, "ematch_matches": matched, "rebuild_forced": rb, "rebuild_cascade": cas,
               "greedy": step["greedy"], "costs": step["costs"], "apply_wave": step["apply_wave"],
               "cascade_nodes_after": nodes_after, "total_cost": res.total_cost}
        for k, v in cur.items():
            if isinstance(v, dict) and v["ms"] > 0:
                if k not in best or v["ms"] < best[k]["ms"]:
                    best[k] = v
            else:
                out[k] = v
        del eg, costs, res, filt
    for k, v in best.items():
        v["GBps"] = v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] else 0.0
        v["frac"] = v["GBps"] / peak
        out[k] = v
    out["enodes_matched_per_s"] = 13 * out["nodes"] / (out["ematch_13"]["ms"] / 1e3)
    out["peak_GBps"] = peak
    return out


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1415
    print(json.dumps(run(n, reps=int(os.environ.get("REPS", "3"))), indent=1))
