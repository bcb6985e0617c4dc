#!/usr/bin/env python
"""Summarise an `ncu --set full` report into a markdown table (per launch).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_ncu_full.md

Columns: duration, DRAM bytes read+write (= bench.py's roofline `traffic`),
achieved DRAM GB/s, DRAM % of peak, SM %, FP64 pipe %, warps active %,
registers/thread.
"""
import csv
import io
import subprocess
import sys

COLS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "MB rd"),
    ("dram__bytes_write.sum", "MB wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps %"),
    ("launch__registers_per_thread", "regs"),
]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {k: hdr.index(k) for k, _ in COLS if k in hdr}
    kn = hdr.index("Kernel Name")
    print(f"ncu --set full summary of `{path}`\n")
    print("| kernel | " + " | ".join(h for _, h in COLS) + " | DRAM GB/s |")
    print("|---" * (len(COLS) + 2) + "|")
    for d in data:
        vals = {}
        for k, _ in COLS:
            if k not in ix:
                vals[k] = float("nan")
                continue
            v = float(d[ix[k]].replace(",", ""))
            vals[k] = v * SCALE.get(units[ix[k]], 1.0)
        t_us = vals["gpu__time_duration.sum"]
        gbs = (vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]) * 1e6 / (t_us * 1e-6) / 1e9
        name = d[kn].split("(")[0].replace("void ", "")
        print(f"| `{name}` | " + " | ".join(f"{vals[k]:.1f}" for k, _ in COLS) + f" | {gbs:.0f} |")


if __name__ == "__main__":
    main(sys.argv[1])
