import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_19911_b200 import B200Device, KeyVector
nb, np_ = 1_000_000, 10_000_000
rng = np.random.Generator(np.random.PCG64(1))
b = KeyVector(rng.integers(0, 2*nb, nb).astype(np.float64), np.arange(nb, dtype=np.uint32))
p = KeyVector(rng.integers(0, 2*nb, np_).astype(np.float64), np.arange(np_, dtype=np.uint32))
d = B200Device()
for i in range(6):
    t = time.perf_counter(); r = d.probe(b, p); print("call", i, (time.perf_counter()-t)*1e3, "ms", r.ledger, file=sys.stderr)
