"""Resident C2 join step: eager launches vs one CUDA-graph replay (tools/, not product)."""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import resident  # noqa: E402

nb, np_ = 1_000_000, 10_000_000
rng = np.random.default_rng(1)
bk = torch.from_numpy(rng.integers(0, 2 * nb, nb).astype(np.float64)).cuda()
pk = torch.from_numpy(rng.integers(0, 2 * nb, np_).astype(np.float64)).cuda()
br = torch.arange(nb, dtype=torch.int32, device="cuda")
pr = torch.arange(np_, dtype=torch.int32, device="cuda")
op, ob = resident.join(bk, br, pk, pr)
cap = op.numel()
out_p = torch.empty(cap, dtype=torch.int32, device="cuda")
out_b = torch.empty(cap, dtype=torch.int32, device="cuda")
m = torch.zeros(1, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def step():
    resident.join_build(bk, br)
    resident.join_probe_async(pk, pr, out_p, out_b, m)


def timeit(fn, reps=30):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts[5:]) * 1e3


for _ in range(5):
    step()
torch.cuda.synchronize()
print(f"eager: {timeit(step):.1f} us")
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
torch.cuda.synchronize()
print(f"graph: {timeit(g.replay):.1f} us  (M={int(m.item()):,})")
assert int(m.item()) == op.numel()
assert torch.equal(out_p[:cap], op) and torch.equal(out_b[:cap], ob)
print("graph replay output identical")
