"""Per-source-line instruction / stall totals of one kernel in an ncu report (profiling helper).

    python tools/ncu_lines.py REPORT LAUNCH_INDEX [N]
"""
import csv, subprocess, sys

rep, idx = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", idx, "--launch-count", "1"], capture_output=True, text=True).stdout
fname, rows, hdr = None, [], None
for rec in csv.reader(out.splitlines()):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].rsplit("/", 1)[-1]
    elif rec[0] == "Line No":
        hdr = rec
    elif hdr and rec[0] not in ("", "Function Name"):
        d = dict(zip(hdr[2:], rec[2:]))
        try:
            rows.append((fname, int(rec[0]), rec[1][:70], int(d.get("Instructions Executed", 0) or 0),
                         int(d.get("Warp Stall Sampling (All Samples)", 0) or 0)))
        except ValueError:
            pass
ti = sum(r[3] for r in rows) or 1
ts = sum(r[4] for r in rows) or 1
print(f"total warp instructions {ti:.3e}, stall samples {ts}")
print("-- by instructions")
for r in sorted(rows, key=lambda r: -r[3])[:n]:
    print(f"{r[0]}:{r[1]:5d} {100*r[3]/ti:5.1f}% inst {100*r[4]/ts:5.1f}% stall  {r[2]}")
print("-- by stall samples")
for r in sorted(rows, key=lambda r: -r[4])[:n]:
    print(f"{r[0]}:{r[1]:5d} {100*r[3]/ti:5.1f}% inst {100*r[4]/ts:5.1f}% stall  {r[2]}")
