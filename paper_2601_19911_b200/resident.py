"""Device-resident entry points over torch CUDA tensors (inputs already in HBM).

PyTorch is only plumbing here (allocation, the current stream, and
torch.distributed in sharded.py); every kernel is libgolp_b200's. Row ids are
carried in int32 tensors and reinterpreted as u32 by the library.
"""

from __future__ import annotations

import ctypes as C
import numbers

import torch

from . import _native


def _lib(t: torch.Tensor):
    """The library with the context of t's device current on this thread."""
    lib = _native.load()
    _native.check(lib.golp_use_device(t.device.index if t.device.index is not None else 0))
    return lib


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _check_cols(keys: torch.Tensor, rows: torch.Tensor) -> None:
    if keys.dtype != torch.float64 or rows.dtype not in (torch.int32, torch.uint32):
        raise ValueError("keys must be float64 and rows int32/uint32 tensors")
    if keys.shape != rows.shape or keys.dim() != 1:
        raise ValueError("keys and rows must be 1-D tensors of equal length")
    if not (keys.is_cuda and rows.is_cuda and keys.is_contiguous() and rows.is_contiguous()):
        raise ValueError("keys and rows must be contiguous CUDA tensors")


def topk(keys: torch.Tensor, rows, k: int, stream=None, want_codes: bool = False):
    """Top-k of device-resident (key, row) columns -> (rows[min(k,n)], codes|None).

    rows is the row-id tensor, or an int `row_base` when the row ids are the
    positions row_base + i (extract_keys's arange, store.py:178-181): then no
    row column is read at all (golp_topk_device_positions).
    codes are the order-preserving u64 key codes (int64 storage) of the winners,
    the input of `merge` for cross-GPU reductions.
    """
    if k < 1:
        raise ValueError("k must be at least 1")
    positions = isinstance(rows, numbers.Integral)
    rows = int(rows) if positions else rows
    if positions:
        if keys.dtype != torch.float64 or keys.dim() != 1 or not (keys.is_cuda and keys.is_contiguous()):
            raise ValueError("keys must be a contiguous 1-D float64 CUDA tensor")
        if rows < 0 or rows + keys.numel() > (1 << 32):
            raise ValueError("row ids row_base + i must fit u32")
    else:
        _check_cols(keys, rows)
    n = keys.numel()
    kk = min(k, n)
    out = torch.empty(kk, dtype=torch.int32, device=keys.device)
    codes = torch.empty(kk, dtype=torch.int64, device=keys.device) if want_codes else None
    lib = _lib(keys)
    oc = codes.data_ptr() if (codes is not None and kk) else 0
    if positions:
        _native.check(lib.golp_topk_device_positions(keys.data_ptr(), n, rows, k, out.data_ptr() if kk else 0, oc,
                                                     _stream(stream)))
    else:
        _native.check(lib.golp_topk_device(keys.data_ptr(), rows.data_ptr(), n, k, out.data_ptr() if kk else 0, oc,
                                           _stream(stream)))
    return out, codes


def merge(codes: torch.Tensor, rows: torch.Tensor, k: int, stream=None, want_codes: bool = False):
    """Exact Top-k of already-encoded candidates (e.g. all-gathered local results)."""
    if k < 1:
        raise ValueError("k must be at least 1")
    n = codes.numel()
    kk = min(k, n)
    out = torch.empty(kk, dtype=torch.int32, device=codes.device)
    oc = torch.empty(kk, dtype=torch.int64, device=codes.device) if want_codes else None
    lib = _lib(codes)
    _native.check(lib.golp_topk_merge_device(codes.data_ptr(), rows.data_ptr(), n, k, out.data_ptr() if kk else 0,
                                             oc.data_ptr() if (oc is not None and kk) else 0, _stream(stream)))
    return out, oc


def join_build(keys: torch.Tensor, rows: torch.Tensor, stream=None) -> None:
    _check_cols(keys, rows)
    _native.check(_lib(keys).golp_join_build_device(keys.data_ptr(), rows.data_ptr(), keys.numel(),
                                                        _stream(stream)))


def _check_positions(keys: torch.Tensor, row_base: int) -> None:
    if keys.dtype != torch.float64 or keys.dim() != 1 or not (keys.is_cuda and keys.is_contiguous()):
        raise ValueError("keys must be a contiguous 1-D float64 CUDA tensor")
    if row_base < 0 or row_base + keys.numel() > (1 << 32):
        raise ValueError("row ids row_base + i must fit u32")


def _probe_sync(lib, keys, rows, op, ob, cap, m, stream) -> int:
    """golp_join_probe_device, or its _positions form when rows is an int row base."""
    if isinstance(rows, numbers.Integral):
        return lib.golp_join_probe_device_positions(keys.data_ptr(), keys.numel(), rows, op.data_ptr(),
                                                    ob.data_ptr(), cap, C.byref(m), _stream(stream))
    return lib.golp_join_probe_device(keys.data_ptr(), rows.data_ptr(), keys.numel(), op.data_ptr(),
                                      ob.data_ptr(), cap, C.byref(m), _stream(stream))


def _check_probe(keys, rows):
    """Validates the probe columns -> rows (an int row base, or the row tensor)."""
    if isinstance(rows, numbers.Integral):
        _check_positions(keys, int(rows))
        return int(rows)
    _check_cols(keys, rows)
    return rows


def join_probe(keys: torch.Tensor, rows, out_probe: torch.Tensor, out_build: torch.Tensor,
               stream=None) -> int:
    """Probe the last built table into caller buffers; returns the match count M.
    rows is the probe row-id tensor, or an int row base when the row ids are the
    positions row_base + i (extract_keys): no row column is read.
    Raises CapacityError (pairs truncated) when M exceeds the buffers."""
    rows = _check_probe(keys, rows)
    cap = min(out_probe.numel(), out_build.numel())
    m = C.c_uint64(0)
    _native.check(_probe_sync(_lib(keys), keys, rows, out_probe, out_build, cap, m, stream))
    return int(m.value)


def join_probe_async(keys: torch.Tensor, rows: torch.Tensor, out_probe: torch.Tensor, out_build: torch.Tensor,
                     matches: torch.Tensor, stream=None) -> None:
    """Enqueue a probe of the last built table without synchronizing; the match
    count lands in `matches` (int64 CUDA tensor of one element). Pairs beyond the
    buffers' capacity are dropped: compare matches with the capacity afterwards.
    rows may be an int row base (positions), as in join_probe."""
    rows = _check_probe(keys, rows)
    cap = min(out_probe.numel(), out_build.numel())
    lib = _lib(keys)
    if isinstance(rows, numbers.Integral):
        _native.check(lib.golp_join_probe_device_positions_async(keys.data_ptr(), keys.numel(), rows,
                                                                 out_probe.data_ptr(), out_build.data_ptr(), cap,
                                                                 matches.data_ptr(), _stream(stream)))
    else:
        _native.check(lib.golp_join_probe_device_async(keys.data_ptr(), rows.data_ptr(), keys.numel(),
                                                       out_probe.data_ptr(), out_build.data_ptr(), cap,
                                                       matches.data_ptr(), _stream(stream)))


def join(bkeys, brows, pkeys, prows, capacity: int | None = None, stream=None):
    """Build + probe -> (probe_rows[M], build_rows[M]) int32 tensors (prows may be an
    int row base: probe row ids = positions)."""
    prows = _check_probe(pkeys, prows)
    join_build(bkeys, brows, stream)
    cap = capacity if capacity is not None else max(pkeys.numel(), 1024)
    while True:
        op = torch.empty(cap, dtype=torch.int32, device=pkeys.device)
        ob = torch.empty(cap, dtype=torch.int32, device=pkeys.device)
        m = C.c_uint64(0)
        lib = _lib(pkeys)
        rc = _probe_sync(lib, pkeys, prows, op, ob, cap, m, stream)
        if rc == _native.GOLP_ERR_CAPACITY:
            cap = int(m.value)
            continue
        _native.check(rc)
        return op[: m.value], ob[: m.value]


def full_sort(keys: torch.Tensor, rows: torch.Tensor, stream=None) -> torch.Tensor:
    """Row ids (int32 storage of u32) by key ascending, equal keys by ascending
    row id -- host_full_sort (pkg/src/golp/host.py:127-130) on the device."""
    _check_cols(keys, rows)
    out = torch.empty(keys.numel(), dtype=torch.int32, device=keys.device)
    _native.check(_lib(keys).golp_full_sort_device(keys.data_ptr(), rows.data_ptr(), keys.numel(),
                                                       out.data_ptr() if keys.numel() else 0, _stream(stream)))
    return out


def set_profiling(on: bool, build_start: bool = True) -> None:
    """Library timing events on/off (golp_set_profiling); build_start=False skips
    the event at a join build's start (probe phase still timed, build not)."""
    _native.check(_native.load().golp_set_profiling((1 if build_start else 2) if on else 0))
