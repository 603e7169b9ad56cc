"""Print `ncu --csv --log-file` metric tables compactly: one line per launch."""
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iid, im, iv = (hdr.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value"))
    launches = {}
    for r in rows[1:]:
        key = (r[iid], r[ik].split("(")[0].replace("scu::<unnamed>::", "").replace("void ", ""))
        launches.setdefault(key, {})[r[im]] = r[iv]
    print("==", path)
    for (lid, name), m in launches.items():
        short = {k.replace("smsp__average_warps_issue_stalled_", "stall_").replace("_per_issue_active.ratio", "")
                  .replace(".avg.pct_of_peak_sustained_active", "%").replace("launch__", "")
                  .replace("gpu__time_duration.sum", "ns").replace("smsp__inst_executed.sum", "inst"): v
                 for k, v in m.items()}
        print(lid, name[:40], " ".join(f"{k}={v}" for k, v in short.items()))
