"""Key metrics of one kernel capture (ncu --set full) as JSON (developer tool).

    python profiles/ncu_key_metrics.py gpurun_out/X.ncu-rep "what was captured" > profiles/Y.json

Issue / pipe utilisation, occupancy, registers, DRAM bytes, the stall reasons (per issued
instruction) and the Instruction Statistics section, from `ncu -i --page raw --csv`.
"""
import csv
import io
import json
import subprocess
import sys

rep, what = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("".join(ln for ln in raw.splitlines(True) if ln.startswith('"')))))
hdr, units = rows[0], rows[1]
out = {"report": rep.split("/")[-1], "captured": what, "kernels": []}
KEYS = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"]
for r in rows[2:]:
    k = {}
    for key in KEYS:
        if key in hdr:
            i = hdr.index(key)
            k[key] = [r[i], units[i]] if units[i] else r[i]
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                v = float(r[i])
            except ValueError:
                continue
            if v >= 0.02:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
    k["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    out["kernels"].append(k)
# the Instruction Statistics section (executed / issued instruction totals)
mix_raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv", "--section", "InstructionStats"],
                         capture_output=True, text=True).stdout
out["instruction_stats_section"] = [ln for ln in mix_raw.splitlines() if ln.startswith('"')][:40]
print(json.dumps(out, indent=1))
