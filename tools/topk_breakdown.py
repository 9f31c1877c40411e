"""Device-time breakdown of the resident Top-K pipeline (threshold / filter / select)."""
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import _native, resident  # noqa: E402

for n, k in [(1_000_000, 100), (10_000_000, 100), (100_000_000, 1000)]:
    keys = torch.from_numpy(np.random.Generator(np.random.PCG64(7)).integers(0, 2**53, n).astype(np.float64)).cuda()
    rows = torch.arange(n, dtype=torch.int32, device="cuda")
    resident.set_profiling(True)
    ts, parts = [], []
    for i in range(20):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        resident.topk(keys, rows, k)
        e1.record()
        e1.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1))
            kt = _native.kernel_times()
            parts.append((kt["topk_threshold_ms"], kt["topk_filter_ms"], kt["topk_select_ms"], kt["topk_candidates"]))
    resident.set_profiling(False)
    med = lambda i: statistics.median(p[i] for p in parts)  # noqa: E731
    print(f"n={n:>11,} k={k:>5}: step {statistics.median(ts)*1e3:8.1f} us | threshold {med(0)*1e3:7.1f} "
          f"filter {med(1)*1e3:7.1f} select {med(2)*1e3:7.1f} us | candidates {int(med(3))}")
