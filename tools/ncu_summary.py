"""Summarise one kernel of an ncu report (raw page) into a small JSON for profiles/.
usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json"""
import csv, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__cycles_elapsed.avg.per_second"]
res = {}
for w in want:
    if w in h:
        i = h.index(w)
        res[w] = v[i] + (" " + units[i] if units[i] else "")
stalls = {}
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
        try:
            val = float(v[i])
        except ValueError:
            continue
        if val > 0:
            stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = val
res["stall_samples"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
