"""Summarise an `ncu --csv --log-file` launch list: per-kernel count, mean, total."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = defaultdict(list)
other = defaultdict(dict)
for r in rows[1:]:
    name = r[ik].split("(")[0].replace("scu::<unnamed>::", "")[:48]
    if r[im] == "gpu__time_duration.sum":
        agg[name].append(float(r[iv].replace(",", "")))
    else:
        other[name][r[im]] = r[iv]
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    extra = " ".join(f"{m.split('.')[0].split('__')[-1]}={val}" for m, val in other[k].items())
    print(f"{k:48s} n={len(v):4d} mean={sum(v)/len(v)/1e3:9.1f}us total={sum(v)/1e6:8.2f}ms "
          f"share={sum(v)/tot*100:5.1f}% {extra}")
