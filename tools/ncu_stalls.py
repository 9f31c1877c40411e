"""Stall-reason split, headline counters and the hottest SASS lines of one kernel in an ncu report.
python tools/ncu_stalls.py report.ncu-rep [top_n] [kernel-name regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
kfilt = ["-k", f"regex:{sys.argv[3]}"] if len(sys.argv) > 3 else []


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


raw = subprocess.run(["ncu", "-i", rep, *kfilt, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
d = dict(zip(r[0], r[2]))
stalls = {k: num(v) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
tot = sum(stalls.values()) or 1
print("kernel", d.get("Kernel Name", "")[:80])
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
          "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
          "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]:
    print(f"  {k} = {d.get(k)}")
for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):22s} {100 * v / tot:5.1f}%")
sass = subprocess.run(["ncu", "-i", rep, *kfilt, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                      text=True).stdout
r = list(csv.reader(io.StringIO(sass)))
h = r[1]
rows = [dict(zip(h, x)) for x in r[2:]]
S = "Warp Stall Sampling (All Samples)"
tot = sum(num(x[S]) for x in rows) or 1
print(f"  SASS lines: {len(rows)}")
for i, x in sorted(enumerate(rows), key=lambda ix: -num(ix[1][S]))[:top]:
    print(f"  [{i:5d}] {100 * num(x[S]) / tot:5.1f}%  exec {int(num(x['Instructions Executed'])):9d}  {x['Source'][:90]}")
