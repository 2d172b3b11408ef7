"""Summarise an ncu --set full report into profiles/ (markdown + per-kernel DRAM traffic json).

usage: python profiles/summarize_ncu.py gpurun_out/prof_rN.ncu-rep profiles/rN_ncu_summary.md \
           [rows_per_launch] [source description]

With rows_per_launch (the real state rows of the captured iteration, e.g. bench.py's rows / K of
the same command), profiles/ncu_traffic.json gets per kernel {dram_bytes, rows, duration_us,
source} so bench.py can set roofline.traffic and compare traffic per row with the algorithmic
bytes per row.
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_%"),
    ("FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("smsp__inst_executed.sum", "instructions"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main(rep, out_md, rows_per_launch=None, source=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary of `{os.path.basename(rep)}`", "",
             "| kernel | " + " | ".join(n for _, n in METRICS) + " | top stalls |",
             "|---|" + "---|" * (len(METRICS) + 1)]
    traffic = {}
    for r in data:
        name = r[idx["Kernel Name"]]
        import re
        m = re.search(r"(k_\w+)", name)
        short = m.group(1) if m else name[:40]
        vals = []
        for m, _ in METRICS:
            v = r[idx[m]] if m in idx else ""
            u = units[idx[m]] if m in idx else ""
            vals.append(f"{v} {u}".strip())
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(stalls, reverse=True)[:3])
        lines.append(f"| {short} | " + " | ".join(vals) + f" | {top} |")

        def mbytes(m):
            v = float(r[idx[m]].replace(",", ""))
            u = units[idx[m]]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        t = mbytes("dram__bytes_read.sum") + mbytes("dram__bytes_write.sum")
        dur = float(r[idx["gpu__time_duration.sum"]].replace(",", ""))
        dur *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(
            units[idx["gpu__time_duration.sum"]], 1.0)
        traffic.setdefault(short, []).append((t, dur))
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    if os.environ.get("NCU_NO_TRAFFIC"):  # secondary configs: keep the headline's traffic record
        print("\n".join(lines))
        return
    tj = os.path.join(os.path.dirname(out_md), "ncu_traffic.json")
    with open(tj, "w") as f:
        json.dump({k: {"dram_bytes": sum(x for x, _ in v) / len(v), "duration_us": sum(d for _, d in v) / len(v),
                       "launches": len(v), "rows": rows_per_launch, "source": source or os.path.basename(rep)}
                   for k, v in traffic.items()}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None,
         sys.argv[4] if len(sys.argv) > 4 else None)
