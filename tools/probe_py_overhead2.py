"""Fine split of B200Device.probe's host-side steps at C2 (tools/)."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import B200Device, KeyVector, _native  # noqa: E402
from paper_2601_19911_b200.device import _columns, _result_array  # noqa: E402

nb, np_ = 1_000_000, 10_000_000
rng = np.random.Generator(np.random.PCG64(1))
b = KeyVector(rng.integers(0, 2 * nb, nb).astype(np.float64), np.arange(nb, dtype=np.uint32))
p = KeyVector(rng.integers(0, 2 * nb, np_).astype(np.float64), np.arange(np_, dtype=np.uint32))
d = B200Device()
for _ in range(5):
    d.probe(b, p)
lib = d._lib
T = {k: [] for k in ("cols+touch", "alloc", "set_dense", "c_call", "ledger_total", "wrap", "free")}
for _ in range(20):
    t0 = time.perf_counter()
    bk, br = _columns(b)
    pk, pr = _columns(p)
    for a in (bk, br, pk, pr):
        d.pins.touch(a)
    t1 = time.perf_counter()
    cap = np_ + 1024
    out_p = _result_array(cap)
    out_b = _result_array(cap)
    t2 = time.perf_counter()
    m = C.c_uint64(0)
    led = _native.Ledger()
    lib.golp_set_dense_rows(1)
    t3 = time.perf_counter()
    lib.golp_probe(_native.ptr(bk), _native.ptr(br), nb, _native.ptr(pk), _native.ptr(pr), np_, 0, 0,
                   _native.ptr(out_p), _native.ptr(out_b), cap, C.byref(m), C.byref(led))
    t4 = time.perf_counter()
    x, y = out_p[: m.value], out_b[: m.value]
    t5 = time.perf_counter()
    del x, y, out_p, out_b
    t6 = time.perf_counter()
    for k, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, led.t_h2d + led.t_kernel + led.t_d2h, t5 - t4, t6 - t5)):
        T[k].append(v * 1e6)
for k, v in T.items():
    print(f"{k:12s} median {np.median(v):9.1f} us")
