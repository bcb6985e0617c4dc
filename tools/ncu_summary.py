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
ATOM = [
    ("l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", "RED req L1"),
    ("lts__t_requests_srcunit_tex_op_red.sum", "RED req L2"),
    ("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_red.sum.pct_of_peak_sustained_elapsed", "RED L1 pipe %"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum", "ATOM req L1"),
    ("lts__t_requests_srcunit_tex_op_atom_dot_alu.sum", "ATOM req L2"),
    ("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_atom.sum.pct_of_peak_sustained_elapsed", "ATOM L1 pipe %"),
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
    atom_cols = [c for c in ATOM if c[0] in hdr]
    if not atom_cols:
        return
    print("\n## Atomic / reduction traffic per launch (RED = no return value, ATOM = returning)\n")
    print("| kernel | us | " + " | ".join(h for _, h in atom_cols) + " |")
    print("|---" * (len(atom_cols) + 2) + "|")
    for d in data:
        red = [float(d[hdr.index(k)].replace(",", "")) for k, _ in atom_cols]
        if not any(red):
            continue
        t_us = float(d[ix["gpu__time_duration.sum"]]) * SCALE.get(units[ix["gpu__time_duration.sum"]], 1.0)
        name = d[kn].split("(")[0].replace("void ", "")
        print(f"| `{name}` | {t_us:.1f} | " + " | ".join(
            f"{v:.2f}" if "pct" in k else f"{v:,.0f}" for v, (k, _) in zip(red, atom_cols)) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
