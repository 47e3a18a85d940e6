"""Instruction share and SIMT width per source region of an ncu --set full report of K2
(--import-source on): usage ncu_regions.py <report.ncu-rep> [top N lines]."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + (sys.argv[3] if len(sys.argv) > 3 else "traverse_kernel")], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, th, st, src = collections.Counter(), collections.Counter(), collections.Counter(), {}
cur = None
ix = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        ix = {}
        for i, k in enumerate(r):
            ix.setdefault(k, i)
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue

    def f(k):
        try:
            return float(r[ix[k]].replace(",", ""))
        except (KeyError, ValueError):
            return 0.0
    key = (cur, ln)
    agg[key] += f("Instructions Executed")
    th[key] += f("Thread Instructions Executed")
    st[key] += f("Warp Stall Sampling (All Samples)")
    src[key] = r[1]
tot = sum(agg.values())
tst = sum(st.values()) or 1
# regions: the enclosing __device__ function of each intersect.cu / fiber_device.cuh line
funcs = {}
for fn in ("intersect.cu", "fiber_device.cuh"):
    path = f"paper_1811_03374_b200/csrc/{fn}"
    cur_f = "?"
    for i, line in enumerate(open(path), 1):
        m = re.match(r"^(?:__device__|__global__)[^(]*?(\w+)\(", line)
        if m:
            cur_f = m.group(1)
        funcs[(fn, i)] = cur_f
reg, regt, regs = collections.Counter(), collections.Counter(), collections.Counter()
for k, v in agg.items():
    name = f"{k[0]}:{funcs.get(k, k[0])}"
    reg[name] += v
    regt[name] += th[k]
    regs[name] += st[k]
print(f"total warp instructions {tot:.3g}")
for name, v in reg.most_common(20):
    print(f"{name:40s} inst {100 * v / tot:5.1f}%  simt {regt[name] / max(v, 1):5.1f}  stall-samples {100 * regs[name] / tst:5.1f}%")
print("--- top lines")
for k, v in agg.most_common(top):
    print(f"{k[0][:16]:16s} {k[1]:4d} {100 * v / tot:5.2f}% simt {th[k] / max(v, 1):5.1f} {src[k].strip()[:80]}")
