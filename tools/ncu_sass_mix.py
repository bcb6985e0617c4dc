#!/usr/bin/env python
"""Instruction mix + stall samples per SASS opcode for each kernel of an ncu report.

    python tools/ncu_sass_mix.py REPORT.ncu-rep [kernel-substring] [top-N]
"""
import collections
import csv
import io
import subprocess
import sys


def main(path, sub="", top=25):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    kern, h = None, None
    blocks = []
    for r in rows:
        if r and r[0] == "Kernel Name":
            kern = r[1]
            continue
        if r and r[0] == "Address":
            h = r
            blocks.append((kern, h, []))
            continue
        if blocks and r:
            blocks[-1][2].append(r)
    for kern, h, data in blocks:
        if sub not in kern:
            continue
        si, ei, st = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
        ops, stalls, tot, tst = collections.Counter(), collections.Counter(), 0, 0
        for r in data:
            try:
                n, s = int(r[ei]), int(r[st])
            except (ValueError, IndexError):
                continue
            toks = r[si].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            op = op.split(".")[0]
            ops[op] += n
            stalls[op] += s
            tot += n
            tst += s
        print(f"== {kern[:110]}\n   warp instructions {tot:,}  stall samples {tst:,}")
        for k, v in ops.most_common(int(top)):
            print(f"   {k:10s} {v:12,d} {100 * v / max(tot, 1):5.1f}%   stalls {100 * stalls[k] / max(tst, 1):5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
