"""profiles/sample_kernel_traffic.json from an ncu launch list (DRAM bytes of
the sampling launch group k_sample_v2 + k_deferred_expand + k_deferred_draw,
averaged per launch).  usage: python tools/traffic_json.py launches.csv [config]"""
import csv
import json
import os
import sys
from collections import defaultdict

path = sys.argv[1]
config = sys.argv[2] if len(sys.argv) > 2 else "nytimes"
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ik, iid, im, iv = (hdr.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value"))
per = defaultdict(lambda: defaultdict(dict))
for r in rows[1:]:
    name = r[ik].split("(")[0].split("<")[0].split("::")[-1].replace("void ", "").strip()
    per[name][r[iid]][r[im]] = float(r[iv].replace(",", ""))
group = {"nytimes-fast": ["k_sample_thru"], "nytimes-expected": ["k_expected"]}.get(
    config, ["k_sample_v2", "k_deferred_expand", "k_deferred_draw"])
out = {"_doc": "DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per sampling launch "
               "group (" + " + ".join(group) + "), averaged over the launches in " + path +
               "; bench.py reports it as roofline.traffic.", config: {"source": path}}
total = 0.0
for k in group:
    launches = per.get(k, {})
    if not launches:
        continue
    rd = sum(v.get("dram__bytes_read.sum", 0) for v in launches.values()) / len(launches)
    wr = sum(v.get("dram__bytes_write.sum", 0) for v in launches.values()) / len(launches)
    t = sum(v.get("gpu__time_duration.sum", 0) for v in launches.values()) / len(launches)
    out[config][k] = {"read": int(rd), "write": int(wr), "mean_ns": int(t), "launches": len(launches)}
    total += rd + wr
out[config]["dram_bytes_per_launch"] = int(total)
# merged into profiles/sample_kernel_traffic.json (one entry per bench config)
dst = "profiles/sample_kernel_traffic.json"
try:
    merged = json.load(open(dst))
except (OSError, ValueError):
    merged = {}
merged["_doc"] = ("DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per sampling launch "
                  "group of each bench config, averaged over the launches of its ncu launch list; "
                  "bench.py reports it as roofline.traffic.")
merged[config] = {"kernels": group, **out[config]}
json.dump(merged, open(dst, "w"), indent=1)
print(json.dumps(merged[config], indent=1))
