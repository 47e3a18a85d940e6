"""Summarise an ncu --csv launch list: per kernel name, mean gpu__time_duration (us) and
any other metrics, grouped by consecutive runs."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
by = collections.OrderedDict()
for r in rows[1:]:
    by.setdefault(int(r[ix["ID"]]), [r[ix["Kernel Name"]].split("(")[0], {}])[1][r[ix["Metric Name"]]] = r[ix["Metric Value"]]
group = int(sys.argv[2]) if len(sys.argv) > 2 else 0
names = [v[0] for v in by.values()]
print("launches:", collections.Counter(names))
out = []
for i, (name, m) in by.items():
    out.append((name, {k: float(v.replace(",", "")) for k, v in m.items() if v}))
if group:
    for g in range(0, len(out), group):
        chunk = out[g:g + group]
        agg = collections.OrderedDict()
        for name, m in chunk:
            for k, v in m.items():
                agg.setdefault((name, k), []).append(v)
        print(f"-- group {g // group}")
        for (name, k), vs in agg.items():
            print(f"   {name[-22:]:22s} {k[:50]:50s} {sum(vs)/len(vs):12.2f}")
