"""B200 full sort (host_full_sort, pkg/src/golp/host.py:127-130) parity: reference
golden vectors, then seeded instances against the oracle. Order is compared
exactly (key ascending, -0.0 == +0.0, ties by ascending row id)."""

import numpy as np
import pytest

from golden_io import cases
from oracle import oracle
from paper_2601_19911_b200 import FULL_ROW, KeyVector

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", cases("full_sort"), ids=lambda c: f"{c['tag']}-n{len(c['keys'])}")
def test_full_sort_matches_reference_golden(b200, case):
    res = b200.full_sort(KeyVector(case["keys"], case["rows"]))
    assert res.payload.tolist() == case["expect"].tolist()
    assert res.ledger.h2d_bytes == 12 * len(case["keys"])
    assert res.ledger.d2h_bytes == 4 * len(case["keys"])


def _keys(kind, n, rng):
    if kind == "uniform":
        return rng.integers(0, 2**53, size=n, dtype=np.int64).astype(np.float64)
    if kind == "normal":
        return rng.standard_normal(n)
    if kind == "small_domain":
        v = rng.integers(-3, 4, size=n).astype(np.float64)
        v[rng.random(n) < 0.1] = -0.0
        return v
    if kind == "constant":
        return np.full(n, 2.5)
    if kind == "zipf":
        return np.minimum(rng.zipf(1.2, n), 2**53 - 1).astype(np.float64)
    raise AssertionError(kind)


@pytest.mark.parametrize("kind", ["uniform", "normal", "small_domain", "constant", "zipf"])
@pytest.mark.parametrize("n", [1, 4095, 4096, 4097, 100_000, 1_000_000])
@pytest.mark.parametrize("rows_kind", ["arange", "permuted", "dups"])
def test_full_sort_random_vs_oracle(b200, kind, n, rows_kind):
    rng = np.random.default_rng(n + len(kind) * 7 + len(rows_kind))
    keys = _keys(kind, n, rng)
    if rows_kind == "arange":
        rows = np.arange(n, dtype=np.uint32)
    elif rows_kind == "permuted":
        rows = rng.permutation(n).astype(np.uint32)
    else:  # repeated and large row ids (all four row bytes vary)
        rows = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
        rows[rng.random(n) < 0.3] = 7
    got = b200.full_sort(KeyVector(keys, rows)).payload
    assert np.array_equal(got, oracle.full_sort(keys, rows))


def test_full_sort_empty_and_full_row(b200):
    res = b200.full_sort(KeyVector(np.empty(0), np.empty(0, dtype=np.uint32)))
    assert len(res.payload) == 0 and res.ledger.h2d_bytes == 0
    rng = np.random.default_rng(1)
    kv = KeyVector(rng.standard_normal(50_000), rng.permutation(50_000))
    full = b200.full_sort(kv, mode=FULL_ROW, payload_bytes=188)
    assert np.array_equal(full.payload, oracle.full_sort(kv.keys, kv.rows))
    assert full.ledger.h2d_bytes == 196 * 50_000


def test_full_sort_resident_large(cuda):
    import torch

    from paper_2601_19911_b200 import _native, resident

    n = 20_000_000
    rng = np.random.default_rng(9)
    keys = rng.integers(0, 2**53, size=n, dtype=np.int64).astype(np.float64)
    rows = rng.permutation(n).astype(np.uint32)
    resident.set_profiling(True)
    try:
        out = resident.full_sort(torch.from_numpy(keys).to(cuda), torch.from_numpy(rows.view(np.int32)).to(cuda))
        kt = _native.kernel_times()
    finally:
        resident.set_profiling(False)
    got = out.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, oracle.full_sort(keys, rows))
    assert 8 <= kt["full_sort_passes"] <= 12
