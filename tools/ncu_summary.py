"""Summarise an ncu --set full report of the scoring kernel.

    python tools/ncu_summary.py REPORT.ncu-rep [KERNEL_SOURCE.cuh] [n_items]

Prints the headline metrics (time, DRAM bytes, issue activity, warps,
registers, spills, stall reasons per issue) and the SASS instruction /
stall-sample split per kernel phase (phases are delimited by the
"// ---- <name>" banner comments of the kernel source).
"""
import csv
import io
import os
import re
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sass__inst_executed_register_spilling", "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def raw_metrics(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units, vals = rows[0], rows[1], rows[2]
    return {m: (vals[h.index(m)], units[h.index(m)]) for m in METRICS if m in h}


def phases_of(src_path):
    marks = []
    for i, line in enumerate(open(src_path), 1):
        m = re.search(r"// ---- ([A-Za-z0-9]+)", line)
        if m:
            marks.append((i, m.group(1)))
    return marks


# Inlined helpers are reported at their own source lines; attribute them to
# the kernel phase that calls them (the item phases are banner-delimited).
HELPER_PHASE = {"v6_apply": "P3", "v6_apply_m": "P3", "v6_cached_tokens": "P0",
                "v6_qc": "P2", "v6_qc_value": "P2", "v6_div1000": "P4", "v6_div": "P4"}


def helpers_of(src_path):
    """(first line, last line, phase) of each helper function of the kernel
    source that HELPER_PHASE names."""
    lines = open(src_path).read().split("\n")
    starts = []
    for i, line in enumerate(lines, 1):
        m = re.match(r"\s*__device__.*?\b(v6_\w+)\s*\(", line)
        if m:
            starts.append((i, m.group(1)))
    out = []
    for k, (ln, name) in enumerate(starts):
        end = starts[k + 1][0] - 1 if k + 1 < len(starts) else len(lines)
        if name in HELPER_PHASE:
            out.append((ln, end, HELPER_PHASE[name]))
    return out


def per_line(rep):
    text = ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass")
    agg = defaultdict(lambda: [0.0, 0.0])
    fname, hdr, cur = None, None, None
    for r in csv.reader(io.StringIO(text)):
        if not r:
            continue
        if r[0] == "File Path":
            fname, hdr = os.path.basename(r[1]), None
            continue
        if r[0] == "Line No":
            hdr = r
            i_s = hdr.index("Warp Stall Sampling (All Samples)")
            i_i = hdr.index("Instructions Executed")
            continue
        if hdr is None:
            continue
        if r[0].isdigit():
            cur = (fname, int(r[0]))
        if cur and len(r) > i_i and r[2] and r[2] != "-":
            try:
                agg[cur][0] += float(r[i_s] or 0)
                agg[cur][1] += float(r[i_i] or 0)
            except ValueError:
                pass
    return agg


def main():
    rep = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else None
    n_items = float(sys.argv[3]) if len(sys.argv) > 3 else None
    for k, (v, u) in raw_metrics(rep).items():
        print(f"{k:80s} {v} {u}")
    if not src:
        return
    agg = per_line(rep)
    marks = phases_of(src)
    helpers = helpers_of(src)
    base = os.path.basename(src)
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_i = sum(v[1] for v in agg.values()) or 1
    out = defaultdict(lambda: [0.0, 0.0])
    for (f, line), (s, i) in agg.items():
        name = "helpers:" + f
        if f.startswith("sm_") and "intrinsics" in f:
            name = "warp intrinsics (shfl/ballot/match)"
        if f == base:
            name = "prologue"
            for ln, ph in marks:
                if line >= ln:
                    name = ph
            for a, b, ph in helpers:
                if a <= line <= b:
                    name = ph
                    break
        out[name][0] += s
        out[name][1] += i
    print(f"\nSASS instructions {tot_i:.4g}" + (f" ({tot_i / n_items:.0f} per item)" if n_items else ""))
    for k, (s, i) in sorted(out.items(), key=lambda kv: -kv[1][1]):
        per = f" {i / n_items:7.1f}/item" if n_items else ""
        print(f"  {k:28s} {100 * s / tot_s:5.1f}% samples {100 * i / tot_i:5.1f}% inst{per}")


if __name__ == "__main__":
    main()
