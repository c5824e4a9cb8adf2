"""Summarise the ncu captures of profiles/profile_round.sh into profiles/<round>_ncu_summary.json
and profiles/latest_ncu_summary.json (read by bench.py for roofline.traffic).

    python profiles/summarize_ncu.py r01      # reads gpurun_out/{launches,dram,prof}_r01*
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
R = sys.argv[1] if len(sys.argv) > 1 else "r01"
if R.startswith("-"):
    sys.exit(__doc__)


def read_csv(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    return list(csv.reader(io.StringIO("".join(lines))))


def launches():
    rows = read_csv(os.path.join(OUT, f"launches_{R}.csv"))
    hdr = rows[0]
    iK, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    per = collections.defaultdict(list)
    for r in rows[1:]:
        per[r[iK]].append(float(r[iV]))
    total = sum(sum(v) for v in per.values())
    return {k: {"launches": len(v), "mean_ms": sum(v) / len(v) / 1e6, "max_ms": max(v) / 1e6, "share": sum(v) / total}
            for k, v in per.items()}


def dram():
    rows = read_csv(os.path.join(OUT, f"dram_{R}.csv"))
    hdr = rows[0]
    iM, iU, iV = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}
    d = {r[iM]: float(r[iV].replace(",", "")) * scale.get(r[iU], 1) for r in rows[1:]}
    return d


def hotspots(rep, top=15, kernel=None):
    """Source lines by share of executed warp instructions and of stall samples (of the
    kernels matching `kernel`, an ncu -k filter, when given)."""
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"]
    if kernel:
        cmd[3:3] = ["-k", kernel]
    src = subprocess.run(cmd, capture_output=True, text=True).stdout
    cur, hdr, out = None, None, []
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and r and r[0] and len(r) > 5 and r[2] == "-":
            out.append((int(r[hdr.index("Instructions Executed")] or 0),
                        int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0), f"{cur}:{r[0]}", r[1].strip()[:80]))
    ti = sum(o[0] for o in out) or 1
    ts = sum(o[1] for o in out) or 1
    return [{"line": w, "instr_share": round(i / ti, 4), "stall_share": round(st / ts, 4), "source": src_}
            for i, st, w, src_ in sorted(out, reverse=True)[:top]]


def full(name=None):
    rep = os.path.join(OUT, f"{name or 'prof_' + R}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    # the longest kernel of the capture (the shared-stream capture holds pass 1 and pass 2)
    it = rows[0].index("gpu__time_duration.sum")
    main = max(rows[2:], key=lambda r: float(r[it].replace(",", "") or 0))
    d = {h: (u, v) for h, u, v in zip(rows[0], rows[1], main)}
    d["kernel"] = ("", main[rows[0].index("Kernel Name")]) if "Kernel Name" in rows[0] else ("", "")
    keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__cycles_elapsed.avg.per_second", "kernel",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
            "dram__bytes_write.sum.per_second"]
    keys += [k for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    kname = d["kernel"][1]
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if "eval" in kname:
        cmd[3:3] = ["-k", "regex:eval"]
    src = subprocess.run(cmd, capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    hdr = next(r for r in srows if "Instructions Executed" in r)
    iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
    ops = collections.Counter()
    for r in srows:
        if len(r) > iE and r[iE] and r[iE].isdigit():
            m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", r[iS].strip())
            if m:
                ops[m.group(2)] += int(r[iE])
    tot = sum(ops.values())
    return {k: d[k] for k in keys if k in d}, {k: [v, round(v / tot, 4)] for k, v in ops.most_common(20)}


out = {"round": R, "workload": "cfg3"}
try:
    out["launch_list"] = launches()
    # the bench line's value step is dsi_sim_run + dsi_sim_reduce: the default trial kernel plus the
    # partition check; the trial kernel's share of that step (compare roofline.kernel_share_of_step)
    ll = out["launch_list"]
    trial = [v for k, v in ll.items() if "dsi_trial_kernel<0, 0, 0, 1, 0>" in k]
    check = [v for k, v in ll.items() if "dsi_check_trials_kernel" in k]
    if trial and check:
        t, c = trial[0]["max_ms"], check[0]["mean_ms"]  # (the variant also serves the smaller workloads)
        out["value_step_kernel_share"] = {"trial_kernel_mean_ms": t, "check_kernel_mean_ms": c, "share": t / (t + c)}
except OSError as e:
    out["launch_list_error"] = str(e)
try:
    dd = dram()
    out["full_bench_launch"] = dd
    out["dram_bytes_per_launch"] = dd.get("dram__bytes_read.sum", 0) + dd.get("dram__bytes_write.sum", 0)
except OSError as e:
    out["dram_error"] = str(e)
try:
    # --set full over one full bench launch (cfg3, every config; profiles/profile_round.sh)
    out["set_full"], out["instruction_mix"] = full()
    out["source_hotspots"] = hotspots(os.path.join(OUT, f"prof_{R}.ncu-rep"))
except (OSError, ValueError, IndexError) as e:
    out["full_error"] = str(e)
try:  # the shared-stream kernel on the full cfg3 grid (profiles/profile_round.sh)
    out["set_full_crn"], out["instruction_mix_crn"] = full(f"prof_crn_{R}")
    name = out["set_full_crn"].get("kernel", ("", ""))[1]
    out["source_hotspots_crn"] = hotspots(os.path.join(OUT, f"prof_crn_{R}.ncu-rep"),
                                          kernel="regex:eval" if "eval" in name else None)
except (OSError, ValueError, IndexError) as e:
    out["crn_error"] = str(e)
try:  # the multi-drafter kernel on W.multi_heatmap (profiles/profile_round.sh)
    out["set_full_multi"], out["instruction_mix_multi"] = full(f"prof_multi_{R}")
    out["source_hotspots_multi"] = hotspots(os.path.join(OUT, f"prof_multi_{R}.ncu-rep"))
except (OSError, ValueError, IndexError) as e:
    out["multi_error"] = str(e)
try:  # the means-only passes on the full cfg3 grid (the longer of the two is summarised)
    out["set_full_means"], out["instruction_mix_means"] = full(f"prof_means_{R}")
except (OSError, ValueError, IndexError) as e:
    out["means_error"] = str(e)
for name in (f"{R}_ncu_summary.json", "latest_ncu_summary.json"):
    with open(os.path.join(ROOT, "profiles", name), "w") as f:
        json.dump(out, f, indent=1)
print(json.dumps({k: out.get(k) for k in ("dram_bytes_per_launch", "launch_list")}, indent=1))
