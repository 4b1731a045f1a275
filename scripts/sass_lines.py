"""Map an ncu --page source --print-source sass CSV (one kernel) onto CUDA
source lines using nvdisasm -g of the same cubin.  Usage:
sass_lines.py sass.csv disasm.txt KERNEL_MANGLED [k-th kernel block, default 0]"""
import collections
import csv
import re
import sys

sass, dis, fun = sys.argv[1], sys.argv[2], sys.argv[3]
kidx = int(sys.argv[4]) if len(sys.argv) > 4 else 0
off2line = {}
cur = None
inside = False
for ln in open(dis):
    if ln.startswith("//----") and ".text." in ln:
        inside = ln.strip().endswith(f".text.{fun} --------------------------")
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m and cur:
        off2line[int(m.group(1), 16)] = (cur, m.group(2).strip())
rows = list(csv.reader(open(sass)))
blocks, b = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        b = []
        blocks.append(b)
    elif b is not None and r and r[0].startswith("0x"):
        b.append(r)
hdr = [r for r in rows if r and r[0] == "Address"][0]
ia, ni = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Warp Stall Sampling (Not-issued Samples)")
blk = blocks[kidx]
base = int(blk[0][0], 16)
agg = collections.Counter()
aggn = collections.Counter()
bar = collections.Counter()
tot = 0
for r in blk:
    off = int(r[0], 16) - base
    line, ins = off2line.get(off, ("?", r[1]))
    s = int(r[ia] or 0)
    tot += s
    if ins.startswith("BAR") or "WARPSYNC" in ins:
        bar[line] += s
    else:
        agg[line] += s
        aggn[line] += int(r[ni] or 0)
print(f"total samples {tot}; at barriers {sum(bar.values())}")
print("top barrier lines:", bar.most_common(8))
for line, s in agg.most_common(int(sys.argv[5]) if len(sys.argv) > 5 else 40):
    print(f"{line:24s} {s:7d} {100 * s / max(tot, 1):5.1f}%")
