#!/usr/bin/env python
"""Top source lines by warp-stall samples from an ncu report (all source files of a kernel).

usage: python profiles/ncu_hotlines.py report.ncu-rep [N] [kernel-regex]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
recs = []
fname = "?"
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= si or not r[0] or not r[si]:
        continue
    try:
        recs.append((float(r[si]), float(r[ii] or 0), f"{fname}:{r[0]}", r[1].strip()[:100]))
    except ValueError:
        pass
tot = sum(x[0] for x in recs) or 1
for s, ins, ln, src in sorted(recs, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}% inst={ins:>10.0f}  {ln}: {src}")
