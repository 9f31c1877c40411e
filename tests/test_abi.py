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
