"""Device-resident full sort throughput (tools/, not product).
python tools/sort_bench.py N [arange|permuted]"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import _native, resident  # noqa: E402

n = int(float(sys.argv[1]))
rk = sys.argv[2] if len(sys.argv) > 2 else "arange"
g = torch.Generator(device="cuda").manual_seed(3)
keys = torch.randint(0, 2**53, (n,), device="cuda", generator=g, dtype=torch.int64).double()
rows = torch.arange(n, dtype=torch.int32, device="cuda")
if rk == "permuted":
    rows = rows[torch.randperm(n, device="cuda", generator=g)]
resident.set_profiling(True)
ts = []
for i in range(5):
    out = resident.full_sort(keys, rows)
    torch.cuda.synchronize()
    kt = _native.kernel_times()
    ts.append(kt["full_sort_ms"])
resident.set_profiling(False)
ms = statistics.median(ts[1:])
passes = kt["full_sort_passes"]
print(f"n={n:,} rows={rk}: {ms:.3f} ms, {n / ms / 1e6:.1f} Gkeys/s, passes={passes}, "
      f"{(24 * passes + 12) * n / ms / 1e6:.0f} GB/s moved (24 B/item/pass + 12 B hist)")
