"""Write a compact text summary of an ncu report (--set full) or launch list (--csv) into
profiles/.  Usage: summarize_ncu.py full <report.ncu-rep> <out.txt>
                   summarize_ncu.py launches <launches.csv> <out.txt>"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__inst_issued.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "sm__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_fmul_pred_on.sum",
]


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    ix = {k: i for i, k in enumerate(h)}
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary of {rep}\n")
        for r in rows[2:]:
            f.write(f"\n## {r[ix['Kernel Name']]}\n")
            for m in METRICS:
                if m in ix:
                    f.write(f"{m:80s} {r[ix[m]]:>16s} {units[ix[m]]}\n")


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        v = v / 1e3 if unit == "nsecond" or unit == "ns" else v
        tot[name] += v
        cnt[name] += 1
    allt = sum(tot.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary of {path} (cold-cache, serialised; compare shares)\n")
        f.write(f"{'kernel':60s} {'launches':>9s} {'total us':>12s} {'mean us':>10s} {'share':>7s}\n")
        for name, t in tot.most_common():
            f.write(f"{name:60s} {cnt[name]:9d} {t:12.1f} {t / cnt[name]:10.2f} {t / allt:7.1%}\n")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
