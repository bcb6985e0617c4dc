#!/usr/bin/env python
"""Per-CUDA-source-line warp-stall samples and executed instructions of one
kernel in an ncu report (captured with -lineinfo and --import-source on).

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [top-N]
"""
import csv
import io
import subprocess
import sys


def main(path, kern, top=30):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = None
    lines = []
    fname = "?"
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            hdr = None
            continue
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[0]:
            continue
        d = dict(zip(hdr, r))
        # duplicate "Source" header: first = CUDA source text
        try:
            samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            inst = float(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        lines.append((f"{fname}:{r[0]}", r[1].strip(), samp, inst))
        if len(lines) > 0 and d is None:
            break
    tot_s = sum(x[2] for x in lines) or 1.0
    tot_i = sum(x[3] for x in lines) or 1.0
    print(f"{'line':>24} {'stall%':>7} {'inst%':>7}  source   (total samples {tot_s:.0f}, warp insts {tot_i:.3g})")
    for ln, src, s, i in sorted(lines, key=lambda x: -x[2])[:top]:
        print(f"{ln:>24} {100 * s / tot_s:7.2f} {100 * i / tot_i:7.2f}  {src[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
