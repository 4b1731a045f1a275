"""Warm kernel timeline of one bench step (configs[1] BERT by default) through
torch.profiler (CUPTI activity records of every kernel in the process, our
libtsat.so included): step span, summed kernel time, GPU idle gaps, top
kernels by warm time, and the biggest gaps with the kernels around them.
Usage: trace_step.py [model] [k_multi]"""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_01332_b200 import models  # noqa: E402
from paper_2101_01332_b200.cost import CostModel, egraph_costs  # noqa: E402
from paper_2101_01332_b200.explorer import ExploreLimits, saturate  # noqa: E402
from paper_2101_01332_b200.extract import greedy_extract  # noqa: E402
from paper_2101_01332_b200.rules import default_rules  # noqa: E402
from paper_2101_01332_b200.tensor_lang import build_egraph  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bert"
km = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = models.MODELS[name]()
rules = list(default_rules())


def step():
    eg = build_egraph(g)[0]
    torch.cuda.synchronize()
    return eg


for i in range(3):
    eg = step()
    filt, rep = saturate(eg, rules, ExploreLimits(k_multi=km))
    greedy_extract(eg, egraph_costs(eg, CostModel()), filt)
    torch.cuda.synchronize()
    del eg
eg = step()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    filt, rep = saturate(eg, rules, ExploreLimits(k_multi=km))
    res = greedy_extract(eg, egraph_costs(eg, CostModel()), filt)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev if e.time_range.end > e.time_range.start])
ker = [k for k in ks if "Memcpy" not in k[2] and "Memset" not in k[2]]
span = ks[-1][1] - ks[0][0]
busy = 0
last = ks[0][0]
gaps = []
for a, b, n in ks:
    if a > last:
        gaps.append((a - last, n))
    busy += max(0, b - max(a, last))
    last = max(last, b)
print(f"{name}: span {span / 1e3:.3f} ms, busy {busy / 1e3:.3f} ms, idle {(span - busy) / 1e3:.3f} ms, "
      f"{len(ker)} kernels, {len(ks) - len(ker)} memcpy/memset")
agg = collections.defaultdict(lambda: [0, 0.0])
for a, b, n in ker:
    k = n.split("(")[0][:60]
    agg[k][0] += 1
    agg[k][1] += b - a
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {k:60s} {c:5d} {t / 1e3:8.3f} ms")
gh = collections.Counter()
for d, n in gaps:
    if d > 0:
        gh[n.split("(")[0][:50]] += d
print("idle before (top):")
for k, d in gh.most_common(15):
    print(f"  {k:50s} {d / 1e3:8.3f} ms")
# the biggest single gaps with the operations around them
print("largest gaps:")
last_end, prev = ks[0][0], ""
gl = []
for a, b, n in ks:
    if a > last_end:
        gl.append((a - last_end, prev, n))
    if b > last_end:
        last_end, prev = b, n
for d, p0, n in sorted(gl, reverse=True)[:25]:
    print(f"  {d:8.1f} us  after {p0.split('(')[0][:40]:40s} before {n.split('(')[0][:40]}")
print("gap histogram (us): ", {k: sum(1 for d, _, _ in gl if lo <= d < hi) for k, (lo, hi) in
      {"<5": (0, 5), "5-10": (5, 10), "10-20": (10, 20), "20-50": (20, 50), ">50": (50, 1e9)}.items()},
      "total", round(sum(d for d, _, _ in gl) / 1e3, 3), "ms")
if os.environ.get("TRACE_DUMP"):
    # full timeline (start offset, duration, gap before, name) for offline reading
    with open(os.environ["TRACE_DUMP"], "w") as f:
        t0, last_end = ks[0][0], ks[0][0]
        for a, b, n in ks:
            f.write(f"{(a - t0):10.1f} {b - a:8.1f} {max(0.0, a - last_end):8.1f}  {n.split('(')[0][:70]}\n")
            last_end = max(last_end, b)
