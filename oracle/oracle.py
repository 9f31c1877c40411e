"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of oracle.c, the CPU restatement of
the reference algorithms (see the header of oracle.c for file:line citations).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this
module. The product (paper_2601_19911_b200) never does.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "oracle.c"
LIB = HERE / "liboracle.so"

_lib = None


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        tmp = LIB.with_suffix(".so.tmp")
        subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", str(tmp), str(SRC)], check=True)
        tmp.replace(LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = C.CDLL(str(LIB))
        vp, u64 = C.c_void_p, C.c_uint64
        lib.oracle_mix64.restype = u64
        lib.oracle_mix64.argtypes = [u64]
        lib.oracle_topk.restype = C.c_int64
        lib.oracle_topk.argtypes = [vp, vp, u64, u64, vp]
        lib.oracle_table_capacity.restype = u64
        lib.oracle_table_capacity.argtypes = [u64]
        lib.oracle_hash_build.restype = C.c_int
        lib.oracle_hash_build.argtypes = [vp, vp, u64, u64, vp, vp]
        lib.oracle_hash_probe.restype = u64
        lib.oracle_hash_probe.argtypes = [vp, vp, u64, vp, vp, u64, vp, vp, u64]
        lib.oracle_proxy_topk.restype = C.c_int64
        lib.oracle_proxy_topk.argtypes = [vp, vp, u64, u64, vp, C.c_int]
        lib.oracle_proxy_probe.restype = u64
        lib.oracle_proxy_probe.argtypes = [vp, vp, u64, vp, vp, u64, vp, vp, u64, C.c_int]
        _lib = lib
    return _lib


def _p(a: np.ndarray) -> int:
    return int(a.ctypes.data) if a.size else 0


def _cols(keys, rows):
    return np.ascontiguousarray(keys, dtype=np.float64), np.ascontiguousarray(rows, dtype=np.uint32)


def mix64(v: int) -> int:
    return int(_load().oracle_mix64(v & (2**64 - 1)))


def topk(keys, rows, k: int) -> np.ndarray:
    """host_topk rows (host.py:133-144)."""
    kc, rc = _cols(keys, rows)
    if k < 1:
        raise ValueError("k must be at least 1")
    out = np.empty(min(k, len(kc)), dtype=np.uint32)
    got = _load().oracle_topk(_p(kc), _p(rc), len(kc), k, _p(out))
    assert got == len(out)
    return out


def full_sort(keys, rows) -> np.ndarray:
    """host_full_sort rows (host.py:127-130): np.lexsort((rows, keys)) order --
    key ascending (float compare, so -0.0 ties +0.0), then row id ascending."""
    kc, rc = _cols(keys, rows)
    return rc[np.lexsort((rc, kc))]


def proxy_topk(keys, rows, k: int, workers: int) -> np.ndarray:
    """ProxyDevice.topk answer with `workers` threads (device.py:329-380)."""
    kc, rc = _cols(keys, rows)
    out = np.empty(min(k, len(kc)), dtype=np.uint32)
    got = _load().oracle_proxy_topk(_p(kc), _p(rc), len(kc), k, _p(out), workers)
    assert got == len(out)
    return out


class Table:
    """KeyHashTable with the reference's slot layout (host.py:83-124)."""

    def __init__(self, keys, rows):
        kc, rc = _cols(keys, rows)
        self.capacity = int(_load().oracle_table_capacity(len(kc)))
        self.slot_bits = np.zeros(self.capacity, dtype=np.uint64)
        self.slot_rows = np.full(self.capacity, 0xFFFFFFFF, dtype=np.uint32)
        rc_ = _load().oracle_hash_build(_p(kc), _p(rc), len(kc), self.capacity, _p(self.slot_bits),
                                        _p(self.slot_rows))
        assert rc_ == 0

    def probe(self, keys, rows, workers: int = 1):
        kc, rc = _cols(keys, rows)
        lib = _load()
        args = (_p(self.slot_bits), _p(self.slot_rows), self.capacity, _p(kc), _p(rc), len(kc))
        if workers <= 1:
            m = lib.oracle_hash_probe(*args, 0, 0, 0)
            p = np.empty(m, dtype=np.uint32)
            b = np.empty(m, dtype=np.uint32)
            lib.oracle_hash_probe(*args, _p(p), _p(b), m)
        else:
            cap = max(len(kc), 1)
            while True:
                p = np.empty(cap, dtype=np.uint32)
                b = np.empty(cap, dtype=np.uint32)
                m = lib.oracle_proxy_probe(*args, _p(p), _p(b), cap, workers)
                if m <= cap:
                    return p[:m], b[:m]
                cap = m
        return p, b


def join(build_keys, build_rows, probe_keys, probe_rows):
    """host_hash_probe(host_hash_build(build), probe) as (probe_rows, build_rows)."""
    return Table(build_keys, build_rows).probe(probe_keys, probe_rows)
