"""C1 end to end: B200Device.topk of 1e6 keys from host arrays (pinned after the
2nd call), median of 50 calls, with the ledger phases. --chunk=BYTES sets the pinned
chunk (inputs above chunk/8 keys take the multi-chunk pipeline)."""
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import B200Device, KeyVector  # noqa: E402

rng = np.random.Generator(np.random.PCG64(7))
kv = KeyVector(rng.integers(0, 2**53, size=1_000_000, dtype=np.int64).astype(np.float64),
               np.arange(1_000_000, dtype=np.uint32))
chunk = next((int(float(a.split("=", 1)[1])) for a in sys.argv if a.startswith("--chunk=")), 0)  # pinned chunk bytes
with B200Device(pin_inputs="--nopin" not in sys.argv, pinned_chunk_bytes=chunk) as dev:
    for _ in range(5):
        dev.topk(kv, 100)
    ts, leds = [], []
    for _ in range(50):
        t = time.perf_counter()
        r = dev.topk(kv, 100)
        ts.append(time.perf_counter() - t)
        leds.append(r.ledger)
    mid = sorted(range(50), key=lambda i: ts[i])[25]
    print(f"median {statistics.median(ts) * 1e3:.4f} ms; ledger " +
          " ".join(f"{f}={getattr(leds[mid], f) * 1e3:.4f}" for f in ("t_h2d", "t_kernel", "t_d2h", "t_post")))
