"""Device Top-K latency (n=1e6, k=100, from host arrays) against the idle time
before the call: does the GPU / link slow down after short idle gaps?"""
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import B200Device, random_key_vector  # noqa: E402

kv = random_key_vector(1_000_000, 5)
with B200Device() as dev:
    for _ in range(20):
        dev.topk(kv, 100)
    for gap_ms in (0.0, 0.05, 0.1, 0.25, 0.5, 1.0, 2.0, 5.0):
        ts = []
        for _ in range(60):
            t_end = time.perf_counter() + gap_ms / 1e3
            while time.perf_counter() < t_end:
                pass
            t0 = time.perf_counter()
            dev.topk(kv, 100)
            ts.append(time.perf_counter() - t0)
        ts.sort()
        print(f"gap {gap_ms:5.2f} ms: p50 {statistics.median(ts)*1e3:.4f} ms  p90 {ts[int(0.9*len(ts))]*1e3:.4f} ms")
