"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv --log-file X`) into
the per-kernel table kept under profiles/ (mean ms per launch, share of the step).

    python tools/launch_table.py gpurun_out/launches.csv [STEPS]
"""

from __future__ import annotations

import csv
import re
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    k_name, k_metric, k_val = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    unit_i = h.index("Metric Unit") if "Metric Unit" in h else None
    per = OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= k_val or r[k_metric] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[k_name]).replace("ns2b::tc::", "").replace("ns2b::", "")
        name = name.replace("void ", "")[:58]
        v = float(r[k_val].replace(",", ""))
        unit = r[unit_i] if unit_i is not None else "ns"
        ms = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        per.setdefault(name, []).append(ms)
    step_names = [n for n in per if not n.startswith(("occupancy", "rays"))]
    nsteps = max(len(per[n]) for n in step_names) if step_names else 1
    step = sum(sum(per[n]) for n in step_names) / nsteps
    print(f"{'kernel':58s} launches   mean ms share of step")
    for n, v in per.items():
        share = sum(v) / nsteps / step if n in step_names else float("nan")
        print(f"{n:58s} {len(v):8d} {sum(v) / len(v):9.3f} {share:13.3f}")
    print(f"# step total (sum of per-launch means, excl. the one-off occupancy refresh and bench "
          f"batch sampling): {step:.2f} ms")


if __name__ == "__main__":
    main()
