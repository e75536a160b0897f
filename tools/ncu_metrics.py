"""Headline raw metrics of the four field kernels in an `ncu --set full` capture (profiling helper).

    python tools/ncu_metrics.py REPORT.ncu-rep "header line" > profiles/<tag>_ncu_metrics.txt
"""
import csv
import subprocess
import sys

ROWS = [("ms", "gpu__time_duration.sum", 1.0),
        ("tensor pipe (HMMA subpipe) active %", "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
        ("tc pipe active %", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
        ("smem wavefronts for the tensor core %", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1.0),
        ("issue slots busy %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
        ("L1 throughput %", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
        ("L2 (LTS) throughput %", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
        ("L2 RED sectors % of peak", "lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed", 1.0),
        ("DRAM read (GB)", "dram__bytes_read.sum", None),
        ("DRAM written (GB)", "dram__bytes_write.sum", None)]
NAMES = [("field_gather", "field_gather_kernel"), ("field_fwd2", "field_fwd2_kernel"), ("field_fwd1", "field_fwd_kernel"),
         ("field_bwd2", "field_bwd2_kernel"), ("field_bwd1", "field_bwd_kernel"), ("field_scatter", "field_scatter_kernel")]


def main():
    rep, header = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    kcol = h.index("Kernel Name")
    kern = []
    for r in rows[2:]:
        nm = next((s for s, k in NAMES if r[kcol].split("(")[0].split()[-1].startswith(k) and
                   (r[kcol].split("(")[0].split()[-1].split("<")[0] == k)), r[kcol][:20])
        kern.append((nm, r))
    if header:
        print("# " + header)
    print(f"{'metric':40s}" + "".join(f"{nm:>22s}" for nm, _ in kern))
    for label, key, _ in ROWS:
        i = h.index(key)
        vals = []
        for _, r in kern:
            v = float(r[i].replace(",", "")) if r[i] else float("nan")
            if units[i] == "Mbyte":
                v /= 1e3
            elif units[i] == "Kbyte":
                v /= 1e6
            elif units[i] == "byte":
                v /= 1e9
            elif units[i] == "us":
                v /= 1e3
            elif units[i] == "ns":
                v /= 1e6
            vals.append(v)
        print(f"{label:40s}" + "".join(f"{v:22.6f}" for v in vals))


if __name__ == "__main__":
    main()
