"""Aggregate an ncu 'source --print-source cuda,sass' CSV per CUDA source line.

    ncu -i prof.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]

The export holds one section per source file ("File Path" row, then a
"Line No" header); lines are keyed by (file, line).
"""
import csv
import os
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    agg = defaultdict(lambda: [0.0, 0.0])
    src = {}
    fname = "?"
    hdr = None
    cur = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            hdr = None
            continue
        if r[0] == "Line No":
            hdr = r
            i_samp = hdr.index("Warp Stall Sampling (All Samples)")
            i_inst = hdr.index("Instructions Executed")
            continue
        if hdr is None:
            continue
        if r[0]:
            if r[0].isdigit():
                cur = (fname, int(r[0]))
                src[cur] = r[1]
        if cur is not None and len(r) > i_inst and r[2]:
            try:
                agg[cur][0] += float(r[i_samp] or 0)
                agg[cur][1] += float(r[i_inst] or 0)
            except ValueError:
                pass
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_i = sum(v[1] for v in agg.values()) or 1
    print(f"total samples {tot_s:.0f}  warp-instructions {tot_i:.3e}")
    for key, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        f, line = key
        print(f"{f[:18]:18s}:{line:4d} {100*s/tot_s:5.1f}% samp {100*n/tot_i:5.1f}% inst"
              f" | {src.get(key, '').strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
