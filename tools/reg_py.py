"""Registered numpy columns: raw cudaMemcpyAsync timing from Python (cuda-python),
to separate the memory itself from the library's transfer path."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import cuda.bindings.runtime as rt  # noqa: E402

from paper_2601_19911_b200 import _native, random_key_vector  # noqa: E402

kv = random_key_vector(1_000_000, 7)
lib = _native.load()
lib.golp_init(0, 16 << 20, 4)
_, d = rt.cudaMalloc(12 << 20)
_, s = rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking)
_, ev = rt.cudaEventCreateWithFlags(rt.cudaEventDisableTiming)


def t(tag, a, b):
    ts = []
    for r in range(30):
        t0 = time.perf_counter()
        rt.cudaMemcpyAsync(d, a.ctypes.data, a.nbytes, rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s)
        rt.cudaMemcpyAsync(int(d) + a.nbytes, b.ctypes.data, b.nbytes, rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s)
        rt.cudaEventRecord(ev, s)
        rt.cudaEventSynchronize(ev)
        ts.append(time.perf_counter() - t0)
    print(f"{tag:40s} min {min(ts[5:])*1e3:.3f} ms median {sorted(ts[5:])[12]*1e3:.3f} ms")


print("register:", lib.golp_host_register(kv.keys.ctypes.data, kv.keys.nbytes),
      lib.golp_host_register(kv.rows.ctypes.data, kv.rows.nbytes))
t("numpy registered via lib", kv.keys, kv.rows)
k2 = kv.keys.copy(); r2 = kv.rows.copy()
print(rt.cudaHostRegister(k2.ctypes.data, k2.nbytes, 0), rt.cudaHostRegister(r2.ctypes.data, r2.nbytes, 0))
t("numpy copy registered default", k2, r2)
k3 = _native.host_array(1_000_000, np.float64); k3[:] = kv.keys
r3 = _native.host_array(1_000_000); r3[:] = kv.rows
t("arena", k3, r3)

from paper_2601_19911_b200 import B200Device, KeyVector  # noqa: E402

dev = B200Device()
t("numpy registered, B200Device alive", kv.keys, kv.rows)
for i in range(5):
    dev.topk(KeyVector(k2, r2), 100)
t("after topk calls", kv.keys, kv.rows)
