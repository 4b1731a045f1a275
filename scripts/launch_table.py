"""Summarise an ncu --csv launch list (gpu__time_duration + optional DRAM
bytes): per-kernel totals, or the launches after the last occurrence of a
kernel name.  Usage: launch_table.py file.csv [--after NAME [--count K]]"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) > vi:
            d.setdefault(r[ii], {"name": r[ki].split("(")[0]})[r[mi]] = float(r[vi].replace(",", ""))
    return list(d.values())


def fmt(x):
    return (f"{x['name'][:44]:44s} {x.get('gpu__time_duration.sum', 0) / 1e3:9.1f} us"
            f"  R {x.get('dram__bytes_read.sum', 0) / 1e6:8.1f} MB  W {x.get('dram__bytes_write.sum', 0) / 1e6:7.1f} MB")


if __name__ == "__main__":
    L = load(sys.argv[1])
    if "--after" in sys.argv:
        name = sys.argv[sys.argv.index("--after") + 1]
        k = int(sys.argv[sys.argv.index("--count") + 1]) if "--count" in sys.argv else 20
        idx = [i for i, x in enumerate(L) if name in x["name"]]
        for x in L[idx[-1]:idx[-1] + k]:
            print(fmt(x))
    else:
        agg = collections.defaultdict(lambda: {"n": 0, "t": 0.0})
        for x in L:
            a = agg[x["name"][:60]]
            a["n"] += 1
            a["t"] += x.get("gpu__time_duration.sum", 0)
        tot = sum(a["t"] for a in agg.values())
        for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"])[:30]:
            print(f"{k:60s} {a['n']:6d} {a['t'] / 1e3:10.1f} us {100 * a['t'] / tot:5.1f}%")
