#!/usr/bin/env python
"""Benchmark: explore + extract search time per graph on B200 (BASELINE.json).

Default workload = configs[1]: BERT-base graph (models.bert), all 14 rules,
k_multi=1, N_max=50k, k_max=15, efficient cycle filtering, synthetic cost
model, greedy extraction.  One step = one full explore + egraph_costs +
greedy_extract of one graph (the reference's three timed spans).

Arms:
  * value: device-resident -- the initial e-graph is uploaded before the timed
    region; the step runs saturate + costs + greedy on the GPU.
  * e2e:   the public API from a host TensorGraph (explore -> egraph_costs ->
    greedy_extract), host<->device copies inside the timed region.
  * --impl reference: the CPU port of the reference (oracle/, the reference
    itself is pure Python and cannot travel to the GPU box) on all host cores.
N>1: one process per GPU; by default the ranks search ONE graph together
(e-matching sharded by e-class range, match lists and greedy wide-level
records all-gathered over NCCL; strong scaling); --replicas runs one
independent graph per GPU instead (weak scaling, no collective).
"""

from __future__ import annotations

import argparse
import ctypes as C
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "bert": dict(model="bert", k_multi=1, n_max=50000, k_max=15,
                 desc="configs[1]: BERT-base (12 layers, seq 64, hidden 768), all 14 rules, k_multi=1, "
                      "N_max=50k, k_max=15, efficient cycle filtering, greedy"),
    "nasrnn": dict(model="nasrnn", k_multi=0, n_max=50000, k_max=15,
                   desc="configs[0]: NasRNN, single-pattern rules only, k_max=15, N_max=50k, greedy"),
    "squeezenet": dict(model="squeezenet", k_multi=2, n_max=100000, k_max=15,
                       desc="configs[2]: SqueezeNet, k_multi=2, N_max=100k, greedy"),
    "resnext50": dict(model="resnext50", k_multi=2, n_max=100000, k_max=15,
                      desc="configs[2]: ResNeXt-50, k_multi=2, N_max=100k, greedy"),
    "inception_v3": dict(model="inception_v3", k_multi=2, n_max=50000, k_max=15,
                         desc="configs[3]: Inception-v3, k_multi=2, greedy"),
    "nasnet_a": dict(model="nasnet_a", k_multi=2, n_max=50000, k_max=15,
                     desc="configs[3]: NasNet-A, k_multi=2, greedy"),
    "synth10m": dict(model="synth10m", k_multi=1, n_max=10**9, k_max=1, sample_n=150,
                     desc="configs[4]: matmul_chain(1415) + matmul-merge-shared-lhs, k_multi=1, k_max=1 "
                          "(10,009,713 e-nodes, 6,008,093 classes), efficient filtering, greedy"),
}

L2_NOTE = "flushed (256 MiB write) between steps"
KGROUPS = ["rebuild", "ematch", "apply_seq", "apply_wave", "reach", "cycles", "costs", "greedy", "snapshot"]
KERNEL_OF = {"rebuild": "rebuild round (k_canon_kids+k_dedup_insert+k_dedup_drop)",
             "ematch": "e-match (k_ematch + radix ordering + unique)",
             "greedy": "greedy (k_greedy_levels/_wide + selection BFS)",
             "reach": "descendants bitset (peel + k_close_block/level)", "apply_seq": "k_seq_rule",
             "apply_wave": "wave apply (k_wave_cta single-CTA waves; grid waves: k_gates, k_resolve_level, k_cand_check, k_conflicts_grid, commit kernels)",
             "costs": "k_node_costs", "cycles": "cycle check (peel/BFS/DFS)", "snapshot": "snapshot CSR"}


# source files whose kernels each ncu region describes: a capture whose stored
# sha256 of any of them differs from the tree being benchmarked is stale
NCU_SOURCES = {"ematch_13": ["match.cu", "egraph.cuh", "common.cuh"],
               "rebuild_forced": ["core.cu", "egraph.cuh", "common.cuh", "analysis.cuh"],
               "rebuild_cascade": ["core.cu", "egraph.cuh", "common.cuh", "analysis.cuh"],
               "costs": ["extract.cu", "analysis.cuh"], "greedy": ["extract.cu", "levels.cu"],
               "apply_wave": ["wave.cu", "analysis.cuh", "rulesdev.cuh", "egraph.cuh"]}


def load_ncu():
    """The newest profiles/*_ncu_traffic.json (scripts/ncu_summary.py), each
    region marked stale when its kernel sources changed since the capture."""
    import glob
    import hashlib

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_traffic.json")))
    if not files:
        return {}, None
    d = json.load(open(files[-1]))
    srcs = d.get("_sources_sha256", {})
    csrc = os.path.join(ROOT, "paper_2101_01332_b200", "csrc")
    for k, deps in NCU_SOURCES.items():
        if k not in d:
            continue
        for f in deps:
            try:
                cur = hashlib.sha256(open(os.path.join(csrc, f), "rb").read()).hexdigest()
            except OSError:
                cur = None
            if srcs.get(f) != cur:
                d[k]["stale"] = True
    return d, os.path.relpath(files[-1], ROOT)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def build_workload(name, sample=False):
    from paper_2101_01332_b200 import bench_graphs, models
    from paper_2101_01332_b200.rules import default_rules

    w = WORKLOADS[name]
    if w["model"] == "synth10m":
        rules = [r for r in default_rules() if r.name == "matmul-merge-shared-lhs"]
        return bench_graphs.matmul_chain(w["sample_n"] if sample else 1415), rules, w
    return models.MODELS[w["model"]](), list(default_rules()), w


def _ref_modules():
    """The reference's own package (oracle/_ref/tensorsat, installed there by
    __graft_entry__.build() from /root/reference; test infrastructure that
    travels to the GPU box) when present, else the golden-pinned CPU port."""
    ref = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref, "tensorsat")):
        if ref not in sys.path:
            sys.path.insert(0, ref)
        import tensorsat.cost as rc
        import tensorsat.explorer as rx
        import tensorsat.extract as re_
        import tensorsat.rules as rr
        import tensorsat.tensor_lang as rt

        return "reference", (rx, rc, re_, rr, rt)
    return "port", None


def run_cpu_once(name, sample=True):
    """One explore + egraph_costs + greedy_extract on one host core: the
    reference package itself when installed (kind "reference"), else the port
    (kind "port").  The graph is handed over as tensorgraph v1 text."""
    from paper_2101_01332_b200.tensor_lang import emit_graph

    g, rules, w = build_workload(name, sample=sample)
    kind, mods = _ref_modules()
    if kind == "reference":
        rx, rc, re_, rr, rt = mods
        rg = rt.make_single_rooted(rt.parse_graph(emit_graph(g)))
        names = {r.name for r in rules}
        rrules = [r for r in rr.default_rules() if r.name in names]
        t0 = time.perf_counter()
        eg, filt, rep = rx.explore(rg, rrules, rx.ExploreLimits(n_max=w["n_max"], k_max=w["k_max"],
                                                                k_multi=w["k_multi"]), "efficient")
        costs = rc.egraph_costs(eg, rc.CostModel())
        res = re_.greedy_extract(eg, costs, filt)
        return time.perf_counter() - t0, eg.num_nodes, res.total_cost, kind
    from oracle import tsat_oracle as O
    from paper_2101_01332_b200.cost import CostModel

    t0 = time.perf_counter()
    eg, filt, rep = O.oracle_explore(g, rules, n_max=w["n_max"], k_max=w["k_max"], k_multi=w["k_multi"])
    costs = O.oracle_costs(eg, CostModel())
    sel, total, _ = O.oracle_greedy(eg, costs, filt)
    return time.perf_counter() - t0, eg.num_nodes, total, kind


def _scale_10m(w):
    n = w["sample_n"]
    return (5 * 1415 * 1415 - 1415 + 3) / (5 * n * n - n + 3)


def reference_arm(args):
    """The reference's CPU implementation on the same workload, metric and
    config as the B200 arm: one graph per step (the metric is search time per
    graph; the pure-Python reference is single-threaded by construction, so
    one graph uses one core)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _, _, w = build_workload(args.workload, sample=True)
    times = []
    nodes = total = kind = None
    warm = min(args.warmup, 1)  # CPython has nothing to warm beyond imports; bounds the run
    for i in range(warm + args.steps):
        dt, nodes, total, kind = run_cpu_once(args.workload)
        if i >= warm:
            times.append(dt)
    per_graph = statistics.mean(times)
    sample = "the full graph"
    if "sample_n" in w:
        per_graph *= _scale_10m(w)
        sample = (f"matmul_chain({w['sample_n']}) ({nodes} e-nodes), scaled by e-node count to "
                  f"matmul_chain(1415)")
    src = ("tensorsat (the reference package, oracle/_ref)" if kind == "reference"
           else "the golden-pinned CPU port (oracle/tsat_oracle.py)")
    line = {
        "impl": "reference", "metric": "explore+extract search time (s) per graph", "value": per_graph,
        "unit": "s", "n_gpus": args.gpus, "steps": args.steps, "warmup": warm, "ms_per_step": per_graph * 1e3,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "int32+f64",
        "data": "synthetic (authored model graph, random-free)",
        # the same config dict as the B200 arm (the workload; the L2 flush is the GPU arm's between-step rule)
        "config": {"workload": w["desc"], "graphs_per_step": 1, "l2": L2_NOTE},
        "result": {"final_enodes": nodes, "total_cost": total},
        "cpu_baseline": {"value": per_graph, "unit": "s", "cores": 1, "kind": kind,
                         "sample": f"one explore+egraph_costs+greedy_extract per step on {sample}, {src}, "
                                   f"1 core of {os.cpu_count()}"},
        "e2e": {"value": per_graph, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--workload", default="bert", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the configs[4] 10M-node kernel sweep")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: one independent graph per GPU (weak scaling, no collective) instead of the "
                         "default sharded search")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
        return

    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # fewer GPUs than ranks (a one-GPU box exercising the N>1 path): ranks
    # share devices and exchange over gloo through the engine's host transport
    shared_gpus = world > torch.cuda.device_count()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    # N>1 default: the ranks explore ONE graph together -- e-matching split by
    # e-class range with an NCCL all-gather of the match lists, greedy's wide
    # levels split with an all-gather of {cost, node}
    shard_mode = world > 1 and not args.replicas
    if world > 1:
        import torch.distributed as dist

        if shared_gpus:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared_gpus else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    from paper_2101_01332_b200 import _lib
    from paper_2101_01332_b200.cost import CostModel, egraph_costs
    from paper_2101_01332_b200.explorer import ExploreLimits, explore, saturate
    from paper_2101_01332_b200.extract import greedy_extract
    from paper_2101_01332_b200.tensor_lang import build_egraph, initial_enodes

    lib = _lib.load()
    g, rules, w = build_workload(args.workload)
    limits = ExploreLimits(n_max=w["n_max"], k_max=w["k_max"], k_multi=w["k_multi"])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    # ---- device-resident arm: each step's e-graph is uploaded (into a pooled
    # engine) before its timed region starts
    step_s = []
    wall_s = []
    kst = np.zeros((3, 9))
    last = None
    if not os.environ.get("TSAT_BENCH_NOFREEZE"):
        gc.collect()
        gc.freeze()  # (see the e2e arm)
    with Clocks(local) as clk:
        for i in range(args.warmup + args.steps):
            eg = build_egraph(g, device=local)[0]
            if shard_mode:
                from paper_2101_01332_b200.shard import attach_group, attach_host

                (attach_host if shared_gpus else attach_group)(eg)
            flush.zero_()
            barrier()
            ms = np.zeros(9)
            by = np.zeros(9)
            la = np.zeros(9, np.int64)
            lib.tsat_kernel_stats(eg._h, ms.ctypes.data_as(C.POINTER(C.c_double)),
                                  by.ctypes.data_as(C.POINTER(C.c_double)),
                                  la.ctypes.data_as(C.POINTER(C.c_int64)), 9, 1)
            # device timing: CUDA events on the engine's own stream (every kernel
            # of the step runs there or joins it before greedy's read-back)
            sp = C.c_void_p()
            _lib.check(eg._h, lib.tsat_stream(eg._h, C.byref(sp)))
            est = torch.cuda.ExternalStream(sp.value or 0, device=torch.device("cuda", local))
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            ev0.record(est)
            filt, rep = saturate(eg, rules, limits, "efficient")
            costs = egraph_costs(eg, CostModel())
            res = greedy_extract(eg, costs, filt)
            ev1.record(est)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            dt = ev0.elapsed_time(ev1) / 1e3
            barrier()
            if i >= args.warmup:
                step_s.append(max_over_ranks(dt))
                wall_s.append(max_over_ranks(wall))
                lib.tsat_kernel_stats(eg._h, ms.ctypes.data_as(C.POINTER(C.c_double)),
                                      by.ctypes.data_as(C.POINTER(C.c_double)),
                                      la.ctypes.data_as(C.POINTER(C.c_int64)), 9, 0)
                kst[0] += ms
                kst[1] += by
                kst[2] += la
            last = (eg, rep, res)
            del eg
    clocks = clk.summary()
    eg, rep, res = last
    nodes = rep.enodes_per_iter[-1] if rep.enodes_per_iter else eg.num_nodes
    # the e2e arm's engines come from the same pool as the device arm's
    del eg, last
    # objects alive now (torch, the graph, the device arm's results) move to
    # the permanent generation: a full collection of them (~35 ms with torch
    # loaded) otherwise lands in whichever e2e step crosses the gen-2 threshold
    if not os.environ.get("TSAT_BENCH_NOFREEZE"):
        gc.collect()
        gc.freeze()
    ms_step = statistics.mean(step_s) * 1e3
    value = ms_step / 1e3 / (1 if shard_mode else world)

    # ---- e2e arm through the public API
    ops, kids, _, _ = initial_enodes(g)
    h2d = 4 * len(ops) + 4 * (len(ops) + 1) + 4 * sum(len(k) for k in kids) + 96 * len(ops)
    e2e_s = []
    d2h = 0
    for i in range(args.warmup + args.steps):
        flush.zero_()
        barrier()
        t0 = time.perf_counter()
        eg2, filt2, rep2 = explore(g, rules, limits, "efficient", device=local,
                                   shard_group=True if shard_mode else None)
        costs2 = egraph_costs(eg2, CostModel())
        res2 = greedy_extract(eg2, costs2, filt2)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        barrier()
        if i >= args.warmup:
            e2e_s.append(max_over_ranks(dt))
        # selection (class, node) + the selected nodes' costs + filter ids + rule stats / per-iteration counts
        d2h = (8 * len(res2.selection) + 8 * len(set(res2.selection.values())) + 4 * len(filt2)
               + 8 * 7 * len(rules) + 24 * 15)
        del eg2
    if os.environ.get("TSAT_BENCH_VERBOSE"):
        print("e2e per step (ms):", [round(x * 1e3, 3) for x in e2e_s], "device:",
              [round(x * 1e3, 3) for x in step_s], file=sys.stderr)
    e2e = statistics.mean(e2e_s) / (1 if shard_mode else world)

    # ---- roofline: dominant instrumented kernel group with an algorithmic byte model
    peak, peak_kind = load_peaks()
    per_step = kst / max(len(step_s), 1)
    dom_all = max(range(9), key=lambda i: per_step[0][i])
    with_bytes = [i for i in range(9) if per_step[1][i] > 0]
    dom = dom_all if per_step[1][dom_all] > 0 else (max(with_bytes, key=lambda i: per_step[0][i]) if with_bytes else 0)
    achieved = per_step[1][dom] / (per_step[0][dom] / 1e3) / 1e9 if per_step[0][dom] > 0 else 0.0
    traffic = None
    ncu, ncu_file = load_ncu()
    if w["model"] == "bert" and KGROUPS[dom] in ncu and not ncu[KGROUPS[dom]].get("stale"):
        traffic = ncu[KGROUPS[dom]]["dram_GB"] * 1e9  # per launch, like `achieved`'s launch average
    roofline = {"bound": "hbm", "kernel": KERNEL_OF[KGROUPS[dom]], "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                "launches_per_step": per_step[2][dom], "ms_per_step": per_step[0][dom],
                "algorithmic_bytes_per_step": per_step[1][dom],
                "algorithmic_bytes_per_launch": per_step[1][dom] / max(per_step[2][dom], 1),
                "traffic_source": ncu_file if traffic is not None else None}
    groups_ms = {KGROUPS[i]: round(per_step[0][i], 3) for i in range(9)}

    line = {
        "metric": "explore+extract search time (s) per graph", "value": value, "unit": "s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "timing": "CUDA events on the engine stream, max over ranks; wall clock beside it",
        "wall_ms_per_step": statistics.mean(wall_s) * 1e3,
        "higher_is_better": False, "scaling": "strong" if shard_mode else "weak", "vs_baseline": None,
        "dtype": "int32+f64",
        "data": "synthetic (authored model graph, random-free)",
        "config": {"workload": w["desc"], "graphs_per_step": 1 if shard_mode else world, "l2": L2_NOTE},
        "result": {"final_enodes": nodes, "stop_reason": rep.stop_reason, "total_cost": res.total_cost,
                   "parallelism": f"ematch-shard x{world}" if shard_mode else f"replicas x{world}"},
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "enodes_matched_per_s": None, "kernel_groups_ms_per_step": groups_ms,
        "dominant_group": KGROUPS[dom_all],
        "roofline": roofline, "clocks": clocks, "gpu_launches": int(per_step[2].sum()),
    }
    em_ms = per_step[0][1]
    if em_ms > 0:
        # every live e-node root-tested once per unique canonical pattern
        from paper_2101_01332_b200.rules import canonicalize

        pats_all = {cp.pattern for r in rules for cp in map(canonicalize, r.sources)}
        pats_single = {canonicalize(r.sources[0]).pattern for r in rules if len(r.sources) == 1}
        n0 = len(initial_enodes(g)[0])
        starts = [n0] + rep.enodes_per_iter[:-1]
        tested = sum(n * (len(pats_all) if i < w["k_multi"] else len(pats_single)) for i, n in enumerate(starts))
        line["enodes_matched_per_s"] = tested / (em_ms / 1e3)
    if rank == 0 and (w["model"] == "synth10m" or not args.no_sweep):
        # configs[4] kernel sweep on the 10M-node e-graph: the north star's
        # roofline targets (e-matching and rebuild vs HBM), with the ncu DRAM
        # traffic of the same kernels from the committed captures (profiles/)
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import synth_sweep

        sw = synth_sweep.run(1415, reps=3)
        if w["model"] == "synth10m":
            line["sweep"] = sw
        else:
            def ncu_of(k):
                c = ncu.get(k, {})
                if not c or c.get("stale"):
                    return {"ncu_dram_GB": None, "ncu_dram_GBps": None, "ncu_stale": bool(c)}
                return {"ncu_dram_GB": c.get("dram_GB"), "ncu_dram_GBps": c.get("dram_GBps"),
                        "ncu_kernel_ms": c.get("kernel_ms"), "ncu_dram_over_algorithmic":
                        round(c["dram_GB"] / (sw[k]["bytes"] / 1e9), 3) if sw[k]["bytes"] and "dram_GB" in c
                        and k != "apply_wave" else None}

            line["config5_kernels"] = {
                k: dict({"ms": round(sw[k]["ms"], 4), "algorithmic_GB": round(sw[k]["bytes"] / 1e9, 4),
                         "achieved_GBps": round(sw[k]["GBps"], 1), "frac": round(sw[k]["frac"], 4)},
                        **(ncu_of(k) if k != "apply_wave" else {}))
                for k in ("ematch_13", "rebuild_forced", "rebuild_cascade", "costs", "greedy", "apply_wave") if k in sw}
            line["config5_kernels"]["ncu_capture"] = ncu_file
            line["config5_kernels"]["graph"] = {"nodes": sw["nodes"], "classes": sw["classes"],
                                                "peak_GBps": sw["peak_GBps"],
                                                "enodes_matched_per_s": sw["enodes_matched_per_s"]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        t_cpu, n_cpu, total_cpu, kind = run_cpu_once(args.workload)
        src = "tensorsat, oracle/_ref" if kind == "reference" else "oracle/tsat_oracle.py"
        if "sample_n" in w:
            scale = _scale_10m(w)
            line["cpu_baseline"] = {"value": t_cpu * scale, "unit": "s", "cores": 1, "kind": kind,
                                    "sample": f"matmul_chain({w['sample_n']}) ({n_cpu} e-nodes, {t_cpu:.2f} s on "
                                              f"1 core, {src}) scaled x{scale:.1f} by e-node count"}
        else:
            line["cpu_baseline"] = {"value": t_cpu, "unit": "s", "cores": 1, "kind": kind,
                                    "sample": f"one full explore+costs+greedy of the same graph on 1 core "
                                              f"({src}), {n_cpu} e-nodes, cost {total_cpu:.6f}"}
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
