"""Basic blocks (runs of SASS instructions with equal execution counts) of one kernel in an
ncu --set full report: start address, instructions, executions, average active lanes, share.
Usage: sass_blocks.py <report.ncu-rep> <kernel regex> [min share %]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
mins = float(sys.argv[3]) if len(sys.argv) > 3 else 0.3
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = None
ins = []
for r in rows:
    if r and r[0] == "Address":
        h = {k: i for i, k in enumerate(r)}
        continue
    if h is None or not r or not r[0].startswith("0x"):
        continue
    ex = float(r[h["Instructions Executed"]] or 0)
    th = float(r[h["Thread Instructions Executed"]] or 0)
    st = float(r[h["Warp Stall Sampling (All Samples)"]] or 0)
    ins.append((r[0], r[1].strip(), ex, th, st))
tot = sum(i[2] for i in ins)
tst = sum(i[4] for i in ins) or 1
print(f"# {kern}: {tot:.4g} warp instructions, {len(ins)} SASS instructions")
blocks, cur = [], []
for x in ins:
    if cur and x[2] != cur[-1][2]:
        blocks.append(cur)
        cur = []
    cur.append(x)
if cur:
    blocks.append(cur)
for b in blocks:
    ex = sum(i[2] for i in b)
    if ex / tot * 100 < mins:
        continue
    th = sum(i[3] for i in b)
    st = sum(i[4] for i in b)
    ops = " ".join(i[1].split()[0] for i in b[:6])
    print(f"{b[0][0][-5:]} n={len(b):4d} exec={b[0][2]/1e3:8.1f}k lanes={th/ex:5.1f} share={ex/tot*100:5.1f}% "
          f"stall={st/tst*100:5.1f}%  {ops}")
