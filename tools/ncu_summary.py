"""Key counters of ncu --set full reports -> JSON (profiles/r1_ncu_full_summary.json).
python tools/ncu_summary.py out.json tag=report.ncu-rep [...]"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "lts__t_sectors_srcunit_tex_op_read.sum"]

out = {}
for arg in sys.argv[2:]:
    tag, rep = arg.split("=", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("golp::", "")
        key = f"{tag}:{name}:{d['ID']}"
        out[key] = {m: f"{d[m]} {u.get(m, '')}".strip() for m in METRICS if m in d}
json.dump(out, open(sys.argv[1], "w"), indent=1)
for k, v in out.items():
    print(k, v.get("gpu__time_duration.sum"), "DRAM r/w", v.get("dram__bytes_read.sum"), "/",
          v.get("dram__bytes_write.sum"), "| dram%", v.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"))
