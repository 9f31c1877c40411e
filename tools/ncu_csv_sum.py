"""Mean gpu__time_duration per kernel from an ncu --csv launch list (tools/)."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            agg[d["Kernel Name"].split("(")[0][:40]].append(float(d["Metric Value"].replace(",", "")))
    print(path)
    for k, v in agg.items():
        print(f"  {k:42s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:8.2f} us")
