"""End-to-end C2 (join 1e6 / 1e7) and C1 (Top-K 1e6, K=100) call time per pinned
chunk size: the B200Device staging/upload unit (golp_init's pinned_chunk_bytes).

    python tools/chunk_sweep.py [MiB ...]

Same inputs and call as bench.py's e2e leg; mean of 20 calls after 5 warm-up calls
(the warm-up also page-locks the reused input columns, as in bench.py)."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from bench import WORKLOADS, join_data, topk_data  # noqa: E402
from paper_2601_19911_b200 import B200Device  # noqa: E402
from paper_2601_19911_b200.store import KeyVector  # noqa: E402


def run(dev, fn, warm=5, steps=20):
    ts = []
    for i in range(warm + steps):
        t0 = time.perf_counter()
        fn(dev)
        if i >= warm:
            ts.append(time.perf_counter() - t0)
    return statistics.mean(ts)


def main(mibs):
    bk, br, pk, pr = join_data(WORKLOADS["join_c2"])
    kb, kp = KeyVector(bk, br), KeyVector(pk, pr)
    keys, rows = topk_data(WORKLOADS["topk_c1"])
    kv = KeyVector(keys, rows)
    for mib in mibs:
        dev = B200Device(pinned_chunk_bytes=int(mib * (1 << 20)))
        j = run(dev, lambda d: d.probe(kb, kp))
        t = run(dev, lambda d: d.topk(kv, 100))
        print(f"chunk {mib:6.1f} MiB  C2 e2e {j * 1e3:7.3f} ms  C1 e2e {t * 1e3:7.3f} ms", flush=True)
        dev.close()


if __name__ == "__main__":
    main([float(a) for a in sys.argv[1:]] or [4, 8, 16, 32, 64])
