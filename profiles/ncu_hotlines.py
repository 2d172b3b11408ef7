#!/usr/bin/env python
"""Top source lines by warp-stall samples from an ncu report (source page, cuda view).

usage: python profiles/ncu_hotlines.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
recs = []
for r in rows[hdr_i + 1:]:
    if len(r) <= si or not r[si] or not r[0]:
        continue
    try:
        recs.append((float(r[si]), float(r[ii] or 0), r[0], r[1].strip()[:110]))
    except ValueError:
        pass
tot = sum(x[0] for x in recs) or 1
for s, ins, ln, src in sorted(recs, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}% inst={ins:>10.0f}  L{ln}: {src}")
