"""Late materialization of C2's join pairs (store.materialize_join): 5e6 pairs,
both sides' keys + 188-byte payloads gathered in pair order. Times the native
threaded gather per software-prefetch distance (GOLP_GATHER_PREFETCH, read once per process)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import store  # noqa: E402
from paper_2601_19911_b200.host import ProbeResult  # noqa: E402

nb, np_, m = 1_000_000, 10_000_000, 5_000_000
rng = np.random.default_rng(0)
bt = store.ColumnTable(np.arange(nb, dtype=np.float64), np.full((nb, 188), 7, np.uint8))
pt = store.ColumnTable(np.arange(np_, dtype=np.float64), np.full((np_, 188), 9, np.uint8))
res = ProbeResult(probe_rows=np.sort(rng.integers(0, np_, m).astype(np.uint32)),
                  build_rows=rng.integers(0, nb, m).astype(np.uint32), probe_count=np_)
import os

ts = []
for _ in range(4):
    t = time.perf_counter()
    store.materialize_join(bt, pt, res)
    ts.append(time.perf_counter() - t)
print(f"prefetch {os.environ.get('GOLP_GATHER_PREFETCH', '32'):>3s}: " + " ".join(f"{x * 1e3:.1f}" for x in ts) + " ms")
