"""Aggregate ncu SASS source-page stall samples by opcode / by region (profiling helper)."""
import csv, subprocess, sys, collections, re
"""usage: python tools/sass_hot.py REPORT.ncu-rep [LAUNCH_INDEX|ID:..] [--top]"""
rep, kid = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kid is not None:
    cmd += ["--kernel-id", kid] if ":" in kid else ["--launch-skip", kid, "--launch-count", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
lines = out.splitlines()
i = next(k for k, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(lines[i:]))
h = rows[0]
ix = {n: h.index(n) for n in h}
tot = 0; by_op = collections.Counter(); ni = collections.Counter(); inst = collections.Counter()
seq = []
for r in rows[1:]:
    if len(r) < len(h) or r == h: continue  # repeated header rows (one block per kernel)
    src = r[ix["Source"]].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    n = int(r[ix["Warp Stall Sampling (Not-issued Samples)"]] or 0)
    e = int(r[ix["Instructions Executed"]] or 0)
    tot += s; by_op[op] += s; ni[op] += n; inst[op] += e
    seq.append((r[ix["Address"]], src, s, e))
print("total samples", tot, "instructions", sum(inst.values()))
for op, s in by_op.most_common(25):
    print(f"{op:28s} {s:8d} {100*s/tot:5.1f}%  notissued {ni[op]:8d}  inst {inst[op]:10d}")
if "--top" in sys.argv:
    for a, src, s, e in sorted(seq, key=lambda x: -x[2])[:40]:
        print(f"{a} {s:7d} {e:9d} {src[:90]}")
