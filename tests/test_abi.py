"""The C-ABI library loads, exports exactly what include/golp_b200.h declares,
and its classical host engine (pure CPU code) reproduces the reference."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from golden_io import cases, npz
from paper_2601_19911_b200 import _native
from paper_2601_19911_b200.host import host_hash_build, host_hash_probe, host_topk
from paper_2601_19911_b200.store import KeyVector

HEADER = Path(__file__).resolve().parents[1] / "include" / "golp_b200.h"


def declared_functions() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(golp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("golp_topk", "golp_probe", "golp_probe_copy_out", "golp_init", "golp_shutdown",
                 "golp_topk_device", "golp_join_build_device", "golp_join_probe_device"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    names = declared_functions()
    assert sorted(_native.SIGNATURES) == names
    for name in names:
        assert hasattr(lib, name), name


def test_struct_layouts_match_header():
    assert C.sizeof(_native.Ledger) == 2 * 8 + 4 * 8
    assert C.sizeof(_native.KernelTimes) == 7 * 8 + 6 * 8


def test_version_and_error_string():
    lib = _native.load()
    assert lib.golp_version() == 1
    assert isinstance(_native.last_error(), str)


def test_invalid_arguments_map_to_reference_exceptions():
    lib = _native.load()
    with pytest.raises(ValueError):
        _native.check(lib.golp_host_topk(0, 0, 0, 0, 0, 1))  # k < 1
    with pytest.raises(ValueError):
        _native.check(lib.golp_host_hash_build(0, 0, 0, 12, 0, 0))  # capacity not a power of two


@pytest.mark.parametrize("case", cases("topk"), ids=lambda c: f"{c['tag']}-n{len(c['keys'])}-k{c['k']}")
def test_host_engine_topk_matches_reference(case):
    kv = KeyVector(case["keys"], case["rows"])
    assert host_topk(kv, int(case["k"])).rows.tolist() == case["expect"].tolist()


def test_host_engine_table_layout_matches_reference():
    z = npz("table")
    t = host_hash_build(KeyVector(z["keys"], z["rows"]))
    assert t.capacity == int(z["capacity"])
    assert np.array_equal(t.slot_bits, z["slot_bits"]) and np.array_equal(t.slot_rows, z["slot_rows"])


@pytest.mark.parametrize("case", cases("probe"), ids=lambda c: f"{c['tag']}-{len(c['bkeys'])}x{len(c['pkeys'])}")
def test_host_engine_probe_matches_reference(case):
    res = host_hash_probe(host_hash_build(KeyVector(case["bkeys"], case["brows"])),
                          KeyVector(case["pkeys"], case["prows"]))
    assert res.probe_rows.tolist() == case["exp_p"].tolist()
    assert res.build_rows.tolist() == case["exp_b"].tolist()
    assert res.probe_count == len(case["pkeys"])


@pytest.mark.parametrize("parts,k", [(1, 10), (3, 100), (8, 5_000), (5, 1)])
def test_host_merge_topk_of_shard_lists(parts, k):
    """golp_host_merge_topk (the merge of B200Device(gpus=G)'s per-GPU top-K lists):
    the first k of all lists in host_topk's order -- order code descending, row
    ascending on ties (host.py:141) -- from best-first inputs with ties across lists."""
    from oracle import oracle

    rng = np.random.default_rng(parts * 1000 + k)
    n = 40_000
    keys = rng.integers(-50, 50, n).astype(np.float64)  # heavy ties, negatives, zeros
    rows = rng.permutation(n).astype(np.uint32)
    bounds = np.linspace(0, n, parts + 1).astype(np.int64)
    codes_l, rows_l, counts = [], [], []
    key_of_row = np.empty(n, dtype=np.float64)
    key_of_row[rows] = keys
    for a, b in zip(bounds[:-1], bounds[1:]):
        r = oracle.topk(keys[a:b], rows[a:b], k)  # a shard's best-first list
        kk = key_of_row[r]
        bits = (kk + 0.0).view(np.uint64)
        codes = np.where(bits >> np.uint64(63), ~bits, bits | np.uint64(1 << 63))  # ord(key)
        codes_l.append(codes)
        rows_l.append(r)
        counts.append(len(r))
    codes = np.ascontiguousarray(np.concatenate(codes_l), dtype=np.uint64)
    cand = np.ascontiguousarray(np.concatenate(rows_l), dtype=np.uint32)
    cnt = np.asarray(counts, dtype=np.uint64)
    out = np.empty(k, dtype=np.uint32)
    got = C.c_uint64(0)
    lib = _native.load()
    assert lib.golp_host_merge_topk(_native.ptr(codes), _native.ptr(cand), _native.ptr(cnt), parts, k,
                                    _native.ptr(out), C.byref(got)) == _native.GOLP_OK
    want = oracle.topk(keys, rows, k)
    assert got.value == len(want)
    np.testing.assert_array_equal(out[: got.value], want)


def test_resident_positions_validation_without_gpu():
    """Row bases that would overflow u32 row ids are refused before any device call."""
    import torch

    from paper_2601_19911_b200 import resident

    keys = torch.zeros(10, dtype=torch.float64)
    with pytest.raises(ValueError):
        resident.topk(keys, 0, 3)  # not a CUDA tensor
    with pytest.raises(ValueError):
        resident._check_positions(keys, -1)
    lib = _native.load()
    # u32 overflow is checked first: no context or device is touched
    assert lib.golp_topk_device_positions(None, 10, (1 << 32) - 9, 3, None, None, None) == _native.GOLP_ERR_INVALID
