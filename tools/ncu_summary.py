"""Summarise one kernel of an .ncu-rep (raw page) into JSON with units.

    python tools/ncu_summary.py gpurun_out/prof_contractS_C2.ncu-rep "note" > profiles/x.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
        "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sector_hit_rate.pct",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]

rep, note = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
names, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(names, zip(vals, units)))
out = {"kernel_name": d.get("Kernel Name", ("", ""))[0][:120], "note": note}
for k in KEYS:
    if k in d:
        out[k] = {"value": d[k][0], "unit": d[k][1]}
try:
    busy = float(d["SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg"][0])
    el = float(d["sm__cycles_elapsed.avg"][0])
    out["dmma_pipe_busy_frac_of_elapsed"] = round(busy / el, 4)
except (KeyError, ValueError):
    pass
print(json.dumps(out, indent=1))
