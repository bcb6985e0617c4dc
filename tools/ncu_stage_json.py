#!/usr/bin/env python
"""Write profiles/ncu_<stage>.json for each C3 kernel of an `ncu --set full`
report: DRAM bytes, executed warp instructions, duration and SM clock per
launch (bench.py reports the dominant kernel's as roofline.traffic and
roofline.issue).

    python tools/ncu_stage_json.py REPORT.ncu-rep "SOURCE NOTE"
"""
import csv
import io
import json
import os
import subprocess
import sys

STAGES = [("k_raster<1,", "count_leaves"), ("k_dir_tiles<1,", "scan_leaves"), ("k_dir_tma", "scan_leaves"), ("k_emit<5,", "emit_pofa"),
          ("k_emit_fast<5,", "emit_pofa"), ("k_splat_depth", "splat_depth"), ("k_splat_index_stored", "splat_index"),
          ("k_splat_resolve", "splat_resolve"), ("k_job_setup", "job_setup"), ("k_leaf_fix(", "leaf_order"),
          ("k_leaf_fix_big", "leaf_sort"), ("k_item_scan_expand", "item_expand")]
# atomic / reduction traffic (north star: "atomic throughput"): warp-level
# requests at L1, sectors at L1, requests arriving at L2, and the L1 RED/ATOM
# pipe utilisation
ATOM = {"red_requests_l1": "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
        "red_sectors_l1": "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum",
        "red_requests_l2": "lts__t_requests_srcunit_tex_op_red.sum",
        "red_l1_pipe_pct": "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_red.sum.pct_of_peak_sustained_elapsed",
        "atom_requests_l1": "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum",
        "atom_sectors_l1": "l1tex__t_sectors_pipe_lsu_mem_global_op_atom.sum",
        "atom_requests_l2": "lts__t_requests_srcunit_tex_op_atom_dot_alu.sum",
        "atom_l1_pipe_pct": "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_atom.sum.pct_of_peak_sustained_elapsed"}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path, note):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    col = {n: h.index(n) for n in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                   "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
                                   "smsp__inst_executed.sum")}
    units = rows[1]
    scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
    seen = set()
    for r in rows[2:]:
        name = r[col["Kernel Name"]].replace(" ", "")
        for pat, stage in STAGES:
            if pat.replace(" ", "") in name and stage not in seen:
                seen.add(stage)
                rd = float(r[col["dram__bytes_read.sum"]]) * scale[units[col["dram__bytes_read.sum"]]]
                wr = float(r[col["dram__bytes_write.sum"]]) * scale[units[col["dram__bytes_write.sum"]]]
                out = {"kernel": r[col["Kernel Name"]].split("(")[0], "stage": stage, "source": note,
                       "dram_bytes_per_launch": int(rd + wr),
                       "warp_inst_per_launch": int(float(r[col["smsp__inst_executed.sum"]])),
                       "duration_us_ncu": float(r[col["gpu__time_duration.sum"]]),
                       "sm_ghz_ncu": float(r[col["sm__cycles_elapsed.avg.per_second"]])}
                atoms = {}
                for key, metric in ATOM.items():
                    if metric in h:
                        try:
                            atoms[key] = float(r[h.index(metric)])
                        except ValueError:
                            pass
                if atoms:
                    out["atomics"] = atoms
                with open(os.path.join(ROOT, "profiles", f"ncu_{stage}.json"), "w") as f:
                    json.dump(out, f)
                print(stage, out["dram_bytes_per_launch"], out["warp_inst_per_launch"])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
