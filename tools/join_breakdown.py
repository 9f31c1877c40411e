"""Device-time breakdown of the resident join (build / probe) at a given size.

python tools/join_breakdown.py NB NP DOMAIN [REPS]   (keys uniform in [0, DOMAIN))
Env GOLP_JOIN_SLICE_BYTES / GOLP_JOIN_PART_PROBE select the partitioned path.
"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import _native, resident  # noqa: E402

nb, np_, dom = (int(float(a)) for a in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
g = torch.Generator(device="cuda").manual_seed(1)
bk = torch.randint(0, dom, (nb,), device="cuda", generator=g).double()
pk = torch.randint(0, dom, (np_,), device="cuda", generator=g).double()
br = torch.arange(nb, dtype=torch.int32, device="cuda")
pr = torch.arange(np_, dtype=torch.int32, device="cuda")
cap = np_ + np_ // 2 + 1024
op = torch.empty(cap, dtype=torch.int32, device="cuda")
ob = torch.empty(cap, dtype=torch.int32, device="cuda")
resident.set_profiling(True)
bt, pt = [], []
for i in range(reps + 1):  # the first call (allocations) is dropped
    resident.join_build(bk, br)
    m = resident.join_probe(pk, pr, op, ob)
    kt = _native.kernel_times()
    if i:
        bt.append(kt["join_build_ms"])
        pt.append(kt["join_probe_ms"])
resident.set_profiling(False)
print(f"nb={nb:,} np={np_:,} dom={dom:,} slices={kt['join_slices']} cap={kt['join_capacity']:,} M={m:,}: "
      f"build {statistics.median(bt):.3f} ms probe {statistics.median(pt):.3f} ms")
if "-v" in sys.argv:
    print("  probe ms per rep:", " ".join(f"{x:.3f}" for x in pt))
