"""Summarise a capture_head.sh directory into profiles/<tag>_ncu_traffic.json:
per configs[4] region (all launches inside the profiler window) the summed
kernel time and DRAM bytes; for the BERT step the per-kernel share table and
the wave-apply kernels' DRAM bytes per launch.  The sha256 of every csrc file
at capture time is stored so bench.py can flag a capture older than the code.
Usage: ncu_summary.py gpurun_out/TAG profiles/TAG_ncu_traffic.json"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch_table import load  # noqa: E402

T, B_R, B_W, HIT = "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct"


def region(path, start_at=None):
    """Summed time / DRAM bytes of the launches in a region CSV; start_at = the
    first kernel name prefix that belongs to the group (earlier launches, e.g.
    the snapshot rebuilt after a rule load, are left out)."""
    L = load(path)
    if start_at:
        first = next((i for i, x in enumerate(L) if x["name"].startswith(start_at)), 0)
        L = L[first:]
    t = sum(x.get(T, 0) for x in L) / 1e9
    by = sum(x.get(B_R, 0) + x.get(B_W, 0) for x in L)
    per = collections.OrderedDict()
    for x in L:
        a = per.setdefault(x["name"], {"launches": 0, "us": 0.0, "dram_MB": 0.0})
        a["launches"] += 1
        a["us"] += x.get(T, 0) / 1e3
        a["dram_MB"] += (x.get(B_R, 0) + x.get(B_W, 0)) / 1e6
    for a in per.values():
        a["us"] = round(a["us"], 1)
        a["dram_MB"] = round(a["dram_MB"], 2)
    return {"launches": len(L), "kernel_ms": round(t * 1e3, 4), "dram_GB": round(by / 1e9, 4),
            "dram_GBps": round(by / t / 1e9, 1) if t else None, "kernels": per}


def main(d, out):
    res = {"_source": f"scripts/capture_head.sh -> {d}: ncu --metrics {T},{B_R},{B_W},{HIT} "
                      "--clock-control none --profile-from-start off (one launch list per region; serialised, "
                      "cold-cache per-launch times)"}
    srcs = {}
    for line in open(os.path.join(d, "sources.sha256")):
        h, f = line.split()
        srcs[os.path.basename(f)] = h
    res["_sources_sha256"] = srcs
    for r in ("ematch", "rebuild_forced", "rebuild_cascade", "costs", "greedy"):
        p = os.path.join(d, f"launches_10m_{r}.csv")
        if os.path.exists(p):
            res["ematch_13" if r == "ematch" else r] = region(p, "k_em_" if r == "ematch" else None)
    p = os.path.join(d, "launches_bert.csv")
    if os.path.exists(p):
        b = region(p)
        tot = sum(a["us"] for a in b["kernels"].values())
        for a in b["kernels"].values():
            a["share"] = round(a["us"] / tot, 4) if tot else 0
        b["kernels"] = dict(sorted(b["kernels"].items(), key=lambda kv: -kv[1]["us"]))
        res["bert_step"] = b
        wave = [k for k in b["kernels"] if "k_wave_cta" in k]
        if wave:
            a = b["kernels"][wave[0]]
            res["apply_wave"] = {"kernel": "k_wave_cta (BERT step)", "launches": a["launches"],
                                 "dram_GB": round(a["dram_MB"] / 1e3 / a["launches"], 6),
                                 "dram_GBps": round(a["dram_MB"] / 1e3 / (a["us"] / 1e6), 2) if a["us"] else None}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: (v if not isinstance(v, dict) or "kernels" not in v else
                          {kk: vv for kk, vv in v.items() if kk != "kernels"}) for k, v in res.items()}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
