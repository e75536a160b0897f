"""Summaries of an `ncu --set full` capture of the four field kernels (profiling helper).

    python tools/ncu_summary.py REPORT.ncu-rep OUT_TXT OUT_DRAM_JSON "command line"

OUT_TXT: per-kernel headline metrics (the --page details rows bench.py's roofline cites);
OUT_DRAM_JSON: dram__bytes_read.sum + dram__bytes_write.sum per launch, which bench.py
reads for the roofline `traffic` field.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

NAMES = {"field_gather_kernel": "field_gather", "field_fwd_kernel": "field_mlp_forward", "field_fwd2_kernel": "field_mlp_forward",
         "field_bwd_kernel": "field_mlp_backward", "field_bwd2_kernel": "field_mlp_backward", "field_scatter_kernel": "field_scatter"}
ROWS = ("Memory Throughput", "DRAM Throughput", "Duration", "Compute (SM) Throughput", "Issue Slots Busy",
        "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Block Size", "Grid Size",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy")


def short(name):
    for k, v in NAMES.items():
        if k in name:
            return v
    return None


def main():
    rep, out_txt, out_json, cmd = sys.argv[1:5]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    kn = h.index("Kernel Name")
    rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    dram = {}
    for r in rows[2:]:
        k = short(r[kn])
        if k and k not in dram:
            b_r = float(r[rd].replace(",", "")) * scale[units[rd]]
            b_w = float(r[wr].replace(",", "")) * scale[units[wr]]
            dram[k] = {"dram_read": b_r, "dram_write": b_w, "traffic": b_r + b_w}
    json.dump({"source": f"ncu --set full --clock-control none, c2 workload, one launch each ({cmd})",
               "unit": "bytes per launch", "kernels": dram}, open(out_json, "w"), indent=1)
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    drows = list(csv.reader(io.StringIO(det)))
    dh = drows[0]
    ki, mi, ui, vi = dh.index("Kernel Name"), dh.index("Metric Name"), dh.index("Metric Unit"), dh.index("Metric Value")
    idx_i = dh.index("ID")
    with open(out_txt, "w") as f:
        f.write(f"# {cmd}\n# c2 workload, 1x B200; kernels: gather, MLP forward, MLP backward, table scatter\n")
        seen = set()
        for r in drows[1:]:
            k = short(r[ki])
            if not k or r[mi] not in ROWS or (r[idx_i], r[mi], r[ui]) in seen:
                continue
            seen.add((r[idx_i], r[mi], r[ui]))
            f.write(f"{r[idx_i]:2s} {k:20s} {r[mi]:40s} {r[vi]:>10s} {r[ui]}\n")
        for k, v in dram.items():
            f.write(f"#  {k:20s} DRAM read {v['dram_read'] / 1e9:7.2f} GB  write {v['dram_write'] / 1e9:7.2f} GB "
                    f"per launch\n")


if __name__ == "__main__":
    main()
