#!/usr/bin/env python
"""Print selected `--page details` metrics of one kernel from an ncu report.

    python tools/ncu_details.py REPORT.ncu-rep KERNEL_SUBSTRING [metric-substr ...]
"""
import csv
import io
import subprocess
import sys

DEFAULT = ("Throughput", "Eligible", "Warp Cycles", "Active Warps", "Issued Ipc", "Hit Rate", "Theoretical",
           "Achieved", "Block Limit", "Registers", "Duration")


def main(path, kname, keys):
    raw = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    ki, ni, vi, ui, si = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit",
                                                "Section Name"))
    seen = None
    for row in rows[1:]:
        if kname not in row[ki]:
            continue
        if seen is None:
            seen = row[0]
        if row[0] != seen:
            break
        if any(k in row[ni] for k in keys):
            print(f"{row[si][:28]:28s} | {row[ni][:58]:58s} | {row[vi]} {row[ui]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], tuple(sys.argv[3:]) or DEFAULT)
