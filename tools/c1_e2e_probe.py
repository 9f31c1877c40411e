"""Per-phase ledger of B200Device.topk at C1 (1e6 keys, K=100) from host arrays:
numpy (registered in place after 2 uses) vs pinned-arena copies of the columns."""
import statistics
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402

from paper_2601_19911_b200 import B200Device, KeyVector, _native, random_key_vector  # noqa: E402

kv0 = random_key_vector(1_000_000, 7)
d = B200Device()
lib = _native.load()


def run(kv, tag):
    walls, leds = [], []
    for i in range(40):
        t0 = time.perf_counter()
        r = d.topk(kv, 100)
        walls.append(time.perf_counter() - t0)
        leds.append(r.ledger)
    med = lambda xs: statistics.median(xs[10:]) * 1e3  # noqa: E731
    print(f"{tag:28s} pinned {lib.golp_host_is_pinned(_native.ptr(kv.keys))}{lib.golp_host_is_pinned(_native.ptr(kv.rows))} "
          f"wall {med(walls):.3f} ms  h2d {med([l.t_h2d for l in leds]):.3f}  kernel {med([l.t_kernel for l in leds]):.3f} "
          f" d2h {med([l.t_d2h for l in leds]):.3f}")


ka = _native.host_array(1_000_000, np.float64)
ka[:] = kv0.keys
ra = _native.host_array(1_000_000)
ra[:] = kv0.rows
run(KeyVector(ka, ra), "arena (cudaHostAlloc)")
run(kv0, "numpy (PinCache)")
run(kv0, "numpy (PinCache) again")
run(KeyVector(ka, ra), "arena again")
big = np.empty(1_000_000 + 512, np.float64)
off = (-big.ctypes.data % 4096) // 8
kal = big[off:off + 1_000_000]
kal[:] = kv0.keys
bigr = np.empty(1_000_000 + 1024, np.uint32)
offr = (-bigr.ctypes.data % 4096) // 4
ral = bigr[offr:offr + 1_000_000]
ral[:] = kv0.rows
run(KeyVector(kal, ral), "numpy page-aligned")
