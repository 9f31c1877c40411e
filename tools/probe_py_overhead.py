"""Where the Python-side time of B200Device.probe goes at C2 (tools/)."""
import cProfile
import pstats
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
d = B200Device()
for _ in range(5):
    d.probe(b, p)
over = []
for _ in range(20):
    t = time.perf_counter()
    r = d.probe(b, p)
    wall = time.perf_counter() - t
    over.append(wall - r.ledger.total)
print(f"python-side overhead: median {np.median(over) * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    d.probe(b, p)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
