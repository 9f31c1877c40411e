"""Summarise an ncu --csv launch list: kernel, grid, time (us), DRAM read/write (MB)."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
h = None
launches = OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if not h or len(r) != len(h):
        continue
    d = dict(zip(h, r))
    key = (d["ID"], d["Kernel Name"].split("(")[0], d["Grid Size"])
    launches.setdefault(key, {})[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
tot = 0.0
for (i, name, grid), m in launches.items():
    t = m.get("gpu__time_duration.sum", ("0", "ns"))
    us = float(t[0].replace(",", "")) / (1000.0 if t[1] == "ns" else 1.0 if t[1] == "us" else 1e-3)
    tot += us
    def mb(k):
        if k not in m:
            return ""
        v, u = m[k]
        v = float(v.replace(",", ""))
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)
        return f"{v * scale:10.1f}"
    print(f"{name[:34]:34s} {grid:16s} {us:10.1f} us  rd {mb('dram__bytes_read.sum')} MB  wr {mb('dram__bytes_write.sum')} MB")
print(f"total {tot:.1f} us")
