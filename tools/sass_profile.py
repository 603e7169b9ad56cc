"""Per-opcode and per-block instruction counts from an ncu --set full report
(source page, SASS view).  usage: python tools/sass_profile.py rep.ncu-rep [units]
units = number of work units (e.g. draws/32) to normalise by."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
rows = r[2:]
ia = h.index("Instructions Executed")
isrc = h.index("Source")
ist = h.index("Warp Stall Sampling (All Samples)")


def op_of(src):
    t = src.split()
    return (t[1] if t[0].startswith("@") else t[0]).split(".")[0]


ops = collections.Counter()
stall = collections.Counter()
for x in rows:
    ops[op_of(x[isrc])] += int(x[ia])
    stall[op_of(x[isrc])] += int(x[ist])
tot = sum(ops.values())
print(f"total {tot} = {tot / units:.2f} per unit")
for op, c in ops.most_common(32):
    print(f"{op:10s} {c / units:7.2f}  stall samples {stall[op]}")
if "--blocks" in sys.argv:
    cur, start, n, acc = None, 0, 0, []
    for i, x in enumerate(rows + [["0"] * len(h)]):
        c = int(x[ia])
        if c != cur:
            if cur is not None and cur * n / units > 0.3:
                print(f"{start:5d}-{i - 1:5d} cnt/unit={cur / units:6.3f} n={n:4d} tot/unit={cur * n / units:6.2f}  "
                      + " ".join(acc[:14]))
            cur, start, n, acc = c, i, 0, []
        n += 1
        if i < len(rows):
            acc.append(op_of(x[isrc]))
