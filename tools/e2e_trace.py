"""One traced E2E C2 probe (GOLP_TRACE upload / probe / landing times on stderr)
after warm-up calls; prints the wall times of the untraced calls first."""
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import B200Device, KeyVector  # noqa: E402

nb, np_ = 1_000_000, 10_000_000
rng = np.random.Generator(np.random.PCG64(1))
b = KeyVector(rng.integers(0, 2 * nb, nb).astype(np.float64), np.arange(nb, dtype=np.uint32))
p = KeyVector(rng.integers(0, 2 * nb, np_).astype(np.float64), np.arange(np_, dtype=np.uint32))
dev = B200Device()
ts = []
for i in range(10):
    t0 = time.perf_counter()
    r = dev.probe(b, p)
    ts.append(time.perf_counter() - t0)
print("e2e ms", [round(t * 1e3, 3) for t in ts], "median(3:)", round(statistics.median(ts[3:]) * 1e3, 3), flush=True)
os.environ["GOLP_TRACE"] = "1"
for i in range(2):
    t0 = time.perf_counter()
    r = dev.probe(b, p)
    print(f"traced call {i}: {(time.perf_counter() - t0) * 1e3:.3f} ms ledger h2d {r.ledger.t_h2d*1e3:.3f} "
          f"kern {r.ledger.t_kernel*1e3:.3f} d2h {r.ledger.t_d2h*1e3:.3f} post {r.ledger.t_post*1e3:.3f}", flush=True)
    sys.stderr.flush()
