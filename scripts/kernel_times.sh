#!/bin/bash
# per-kernel device times for fiber A at the given depths (ncu launch list; under gpurun)
python scripts/prof_one.py A 2 > /dev/null || exit 1
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio --clock-control none --csv --log-file gpurun_out/launches_k.csv bash -c "for D in $*; do python scripts/prof_one.py A \$D 1; done" > /dev/null 2>&1
python - "$@" <<'PY'
import csv, collections, sys
rows = [r for r in csv.reader(open("gpurun_out/launches_k.csv")) if len(r) > 10]
h = rows[0]; ix = {k: i for i, k in enumerate(h)}
by = collections.OrderedDict()
for r in rows[1:]:
    by.setdefault(int(r[ix["ID"]]), [r[ix["Kernel Name"]].split("(")[0], {}])[1][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
seq = [v for v in by.values() if "segments" not in v[0]]
depths = sys.argv[1:]
n = len(seq) // len(depths)
for j, D in enumerate(depths):
    agg = collections.defaultdict(list)
    for k, m in seq[j * n:(j + 1) * n]:
        agg[k].append(m)
    print("D=%s " % D + "  ".join("%s %.1fus inst %.3g simt %.1f" % (k.split("::")[-1][:10], sum(m["gpu__time_duration.sum"] for m in ms) / len(ms) / 1e3, sum(m["smsp__inst_executed.sum"] for m in ms) / len(ms), sum(m["smsp__thread_inst_executed_per_inst_executed.ratio"] for m in ms) / len(ms)) for k, ms in agg.items()))
PY
