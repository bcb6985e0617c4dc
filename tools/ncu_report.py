#!/usr/bin/env python
"""Markdown evidence from an `ncu --set full` report: per-kernel table
(tools/ncu_summary.py), issue / occupancy / top stall reasons per kernel, and
the hottest CUDA source lines of the given kernels (tools/ncu_lines.py).

    python tools/ncu_report.py REPORT.ncu-rep "title" [kernel-regex ...] > profiles/X.md
"""
import csv
import io
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
import ncu_lines  # noqa: E402
import ncu_summary  # noqa: E402


def stalls(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    print("| kernel | issue active % | warps active % | top stalls (cycles per issued instruction) |")
    print("|---|---|---|---|")
    for r in rows[2:]:
        d = dict(zip(h, r))
        st = []
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st = [x for x in sorted(st, reverse=True) if x[1] != "selected"][:4]
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("fhv::", "")[:40]
        print(f"| `{name}` | {float(d['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} | "
              f"{float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
              + ", ".join(f"{n} {v:.1f}" for v, n in st) + " |")


def main(path, title, kernels):
    print(f"# {title}\n")
    print(f"Source: `{path}` (`ncu --set full --clock-control none --import-source on`, one launch per row; "
          "per-launch times are cold-cache and serialised -- compare shares, not absolutes).\n")
    sys.stdout.flush()
    ncu_summary.main(path)
    print()
    stalls(path)
    for k in kernels:
        print(f"\n## hottest source lines: `{k}`\n\n```")
        sys.stdout.flush()
        ncu_lines.main(path, k, 15)
        sys.stdout.flush()
        print("```")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3:])
