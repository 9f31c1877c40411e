"""E2E transfer-engine sweep on the GPU box: B200Device.probe / topk wall time for
host-thread counts, pinned chunk sizes and result allocators."""
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import paper_2601_19911_b200.device as D
    from paper_2601_19911_b200 import B200Device, KeyVector, _native

    nb, np_ = 1_000_000, 10_000_000
    rng = np.random.Generator(np.random.PCG64(1))
    b = KeyVector(rng.integers(0, 2 * nb, nb).astype(np.float64), np.arange(nb, dtype=np.uint32))
    p = KeyVector(rng.integers(0, 2 * nb, np_).astype(np.float64), np.arange(np_, dtype=np.uint32))
    for threads in [int(x) for x in sys.argv[1].split(",")]:
        for chunk_mb in [int(x) for x in sys.argv[2].split(",")]:
            for alloc in sys.argv[3].split(","):
                D.RESULT_ALLOCATOR = alloc
                _native.load().golp_shutdown()
                dev = B200Device(pinned_chunk_bytes=chunk_mb << 20, host_threads=threads)
                ts, leds = [], []
                for i in range(8):
                    t0 = time.perf_counter()
                    r = dev.probe(b, p)
                    ts.append(time.perf_counter() - t0)
                    leds.append(r.ledger)
                led = leds[-1]
                print(json.dumps({"threads": threads, "chunk_mb": chunk_mb, "alloc": alloc,
                                  "e2e_ms": statistics.median(ts[3:]) * 1e3,
                                  "h2d": led.t_h2d * 1e3, "kern": led.t_kernel * 1e3, "d2h": led.t_d2h * 1e3,
                                  "post": led.t_post * 1e3}), flush=True)
                dev.close()


if __name__ == "__main__":
    main()
