"""C2 end-to-end probe time for one staging-chunk size (fresh process per size):
    python tools/e2e_chunk_sweep.py CHUNK_MB [host_threads]"""
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import B200Device, KeyVector  # noqa: E402

mb = int(sys.argv[1])
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 0
nb, np_ = 1_000_000, 10_000_000
rng = np.random.Generator(np.random.PCG64(1))
b = KeyVector(rng.integers(0, 2 * nb, nb).astype(np.float64), np.arange(nb, dtype=np.uint32))
p = KeyVector(rng.integers(0, 2 * nb, np_).astype(np.float64), np.arange(np_, dtype=np.uint32))
d = B200Device(pinned_chunk_bytes=mb << 20, host_threads=threads)
ts = []
for i in range(25):
    t = time.perf_counter()
    d.probe(b, p)
    if i >= 5:
        ts.append(time.perf_counter() - t)
print(f"chunk {mb} MB threads {threads}: e2e median {statistics.median(ts) * 1e3:.3f} ms, min {min(ts) * 1e3:.3f} ms")
