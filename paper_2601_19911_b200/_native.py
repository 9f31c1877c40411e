"""ctypes binding of libgolp_b200.so (C ABI in include/golp_b200.h).

The library is the product: there is no Python or CPU fallback for the device
path. If the shared object is missing or fails to load, every device entry
point raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import weakref
from pathlib import Path

import numpy as np

from .errors import CapacityError

LIB_PATH = Path(__file__).resolve().parent / "libgolp_b200.so"

GOLP_OK = 0
GOLP_ERR_INVALID = 1
GOLP_ERR_CAPACITY = 2
GOLP_ERR_CUDA = 3

GOLP_KEY_ONLY = 0
GOLP_FULL_ROW = 1

_vp = C.c_void_p
_u64 = C.c_uint64
_u32 = C.c_uint32
_int = C.c_int


class Ledger(C.Structure):
    _fields_ = [
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("t_h2d", C.c_double),
        ("t_kernel", C.c_double),
        ("t_d2h", C.c_double),
        ("t_post", C.c_double),
    ]


class KernelTimes(C.Structure):
    _fields_ = [
        ("topk_threshold_ms", C.c_double),
        ("topk_filter_ms", C.c_double),
        ("topk_select_ms", C.c_double),
        ("join_build_ms", C.c_double),
        ("join_probe_ms", C.c_double),
        ("topk_candidates", C.c_uint64),
        ("topk_fallback", C.c_uint64),
        ("join_groups", C.c_uint64),
        ("join_capacity", C.c_uint64),
        ("join_slices", C.c_uint64),
        ("full_sort_ms", C.c_double),
        ("full_sort_passes", C.c_uint64),
        ("call_kernel_ms", C.c_double),
    ]


# name -> (restype, argtypes); mirrors include/golp_b200.h one to one
SIGNATURES = {
    "golp_last_error": (C.c_char_p, []),
    "golp_version": (_int, []),
    "golp_init": (_int, [_int, _u64, _int]),
    "golp_use_device": (_int, [_int]),
    "golp_current_device": (_int, [C.POINTER(_int)]),
    "golp_context_open": (_int, [_int, _u64, _int, C.POINTER(_int)]),
    "golp_context_use": (_int, [_int]),
    "golp_context_close": (_int, [_int]),
    "golp_shutdown": (_int, []),
    "golp_launch_count": (_u64, []),
    "golp_last_transfer": (_int, [C.POINTER(_u64), C.POINTER(_u64)]),
    "golp_set_dense_rows": (_int, [_int]),
    "golp_hint_dense_rows": (_int, []),
    "golp_set_profiling": (_int, [_int]),
    "golp_last_kernel_times": (_int, [C.POINTER(KernelTimes)]),
    "golp_topk": (_int, [_vp, _vp, _u64, _u64, _int, _u32, _vp, C.POINTER(_u64), C.POINTER(Ledger)]),
    "golp_topk_codes": (_int, [_vp, _vp, _u64, _u64, _int, _u32, _vp, _vp, C.POINTER(_u64), C.POINTER(Ledger)]),
    "golp_host_merge_topk": (_int, [_vp, _vp, _vp, _int, _u64, _vp, C.POINTER(_u64)]),
    "golp_probe": (_int, [_vp, _vp, _u64, _vp, _vp, _u64, _int, _u32, _vp, _vp, _u64, C.POINTER(_u64),
                          C.POINTER(Ledger)]),
    "golp_probe_copy_out": (_int, [_vp, _vp, _u64, C.POINTER(Ledger)]),
    "golp_topk_device": (_int, [_vp, _vp, _u64, _u64, _vp, _vp, _vp]),
    "golp_topk_device_positions": (_int, [_vp, _u64, _u32, _u64, _vp, _vp, _vp]),
    "golp_topk_merge_device": (_int, [_vp, _vp, _u64, _u64, _vp, _vp, _vp]),
    "golp_join_build_device": (_int, [_vp, _vp, _u64, _vp]),
    "golp_join_probe_device": (_int, [_vp, _vp, _u64, _vp, _vp, _u64, C.POINTER(_u64), _vp]),
    "golp_join_probe_device_async": (_int, [_vp, _vp, _u64, _vp, _vp, _u64, _vp, _vp]),
    "golp_join_probe_device_positions": (_int, [_vp, _u64, _u32, _vp, _vp, _u64, C.POINTER(_u64), _vp]),
    "golp_join_probe_device_positions_async": (_int, [_vp, _u64, _u32, _vp, _vp, _u64, _vp, _vp]),
    "golp_full_sort": (_int, [_vp, _vp, _u64, _int, _u32, _vp, C.POINTER(Ledger)]),
    "golp_full_sort_device": (_int, [_vp, _vp, _u64, _vp, _vp]),
    "golp_host_alloc": (_vp, [_u64]),
    "golp_host_free": (_int, [_vp, _u64]),
    "golp_host_register": (_int, [_vp, _u64]),
    "golp_host_is_pinned": (_int, [_vp]),
    "golp_host_is_pinned_range": (_int, [_vp, _u64]),
    "golp_host_unregister": (_int, [_vp]),
    "golp_host_topk": (_int, [_vp, _vp, _u64, _u64, _vp, _int]),
    "golp_host_hash_build": (_int, [_vp, _vp, _u64, _u64, _vp, _vp]),
    "golp_host_hash_probe": (_int, [_vp, _vp, _u64, _vp, _vp, _u64, _int, C.POINTER(_u64)]),
    "golp_host_probe_copy_out": (_int, [_vp, _vp, _u64]),
    "golp_host_gather": (_int, [_vp, _u64, _u64, _vp, _u64, _vp, _int]),
}

_lib = None


def load() -> C.CDLL:
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("GOLP_B200_LIB", LIB_PATH))
    if not path.exists():
        raise RuntimeError(
            f"{path} is not built: the B200 path has no fallback. "
            "Run `python -c 'import __graft_entry__ as g; g.build()'` first."
        )
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().golp_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int) -> None:
    """Map a golp_status onto the reference's exception types (errors.py)."""
    if rc == GOLP_OK:
        return
    msg = last_error()
    if rc == GOLP_ERR_INVALID:
        raise ValueError(msg)
    if rc == GOLP_ERR_CAPACITY:
        raise CapacityError(msg)
    raise RuntimeError(f"libgolp_b200: {msg}")


def ptr(arr) -> int:
    """Address of a numpy array's first element (0 for empty arrays)."""
    return int(arr.ctypes.data) if arr.size else 0


class _HostBlock:
    """Owner of one golp_host_alloc block; frees it when the last array view dies."""

    __slots__ = ("ptr", "nbytes", "__weakref__")

    def __init__(self, ptr: int, nbytes: int):
        self.ptr = ptr
        self.nbytes = nbytes

    def __del__(self):
        if self.ptr and _lib is not None:
            _lib.golp_host_free(self.ptr, self.nbytes)
            self.ptr = 0


def host_array(n: int, dtype=np.uint32) -> np.ndarray:
    """Fresh 1-D array in library-allocated (huge-page) host memory; the block is
    released when the array and every view of it are gone."""
    dt = np.dtype(dtype)
    nbytes = max(int(n) * dt.itemsize, 1)
    lib = load()
    ptr = lib.golp_host_alloc(nbytes)
    if not ptr:
        raise MemoryError(last_error() or "golp_host_alloc failed")
    owner = _HostBlock(int(ptr), nbytes)
    buf = (C.c_char * nbytes).from_address(int(ptr))
    arr = np.frombuffer(buf, dtype=dt, count=int(n))
    # keep the owner alive as long as any view of the array is
    _keepalive[id(buf)] = owner
    weakref.finalize(buf, _keepalive.pop, id(buf), None)
    return arr


_keepalive: dict = {}


def launch_count() -> int:
    return int(load().golp_launch_count())


def last_transfer() -> tuple:
    """(h2d_bytes, d2h_bytes) the copy engines actually moved during the last
    host-buffer call (a dense row-id column is regenerated on the device, not copied)."""
    h2d, d2h = _u64(0), _u64(0)
    check(load().golp_last_transfer(C.byref(h2d), C.byref(d2h)))
    return int(h2d.value), int(d2h.value)


def kernel_times() -> dict:
    kt = KernelTimes()
    check(load().golp_last_kernel_times(C.byref(kt)))
    return {name: getattr(kt, name) for name, _ in KernelTimes._fields_}
