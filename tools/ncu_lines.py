#!/usr/bin/env python
"""Per-source-line warp-stall sample shares of one kernel in an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [--top N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[3] == "--top" else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
f, agg = None, {}
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) < 5 or r[0] == "Line No" or not r[0]:
        continue
    try:
        s = float(r[4] or 0)
    except ValueError:
        continue
    k = (f, r[0], r[1][:100])
    agg[k] = agg.get(k, 0) + s
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]} {k[2]}")
