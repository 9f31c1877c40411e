"""B200 Top-K parity: golden vectors from the reference, then seeded random
instances against the oracle (bit-exact rows, including tie order)."""

import numpy as np
import pytest

from golden_io import cases
from oracle import oracle
from paper_2601_19911_b200 import FULL_ROW, KeyVector, _native

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", cases("topk"), ids=lambda c: f"{c['tag']}-n{len(c['keys'])}-k{c['k']}")
def test_topk_matches_reference_golden(b200, case):
    kv = KeyVector(case["keys"], case["rows"])
    res = b200.topk(kv, int(case["k"]))
    assert res.backend == "b200"
    assert res.payload.rows.tolist() == case["expect"].tolist()
    assert res.payload.k_requested == int(case["k"])
    assert res.ledger.h2d_bytes == 12 * len(kv)
    assert res.ledger.d2h_bytes == 4 * len(case["expect"])


def _zipf(n, seed, hi):
    r = np.random.default_rng(seed).zipf(1.2, n).astype(np.float64)
    r = np.minimum(r, 2.0**53 - 1)
    return (2.0**53 - 1) - r if hi else r


def _gen(kind, n, rng):
    if kind == "uniform":
        return rng.integers(0, 2**53, size=n, dtype=np.int64).astype(np.float64)
    if kind == "normal":
        return rng.standard_normal(n)
    if kind == "small_domain":
        return rng.integers(-3, 4, size=n).astype(np.float64)
    if kind == "zipf_hi":
        return _zipf(n, int(rng.integers(1 << 30)), True)
    if kind == "zipf_lo":
        return _zipf(n, int(rng.integers(1 << 30)), False)
    if kind == "ascending":
        return np.arange(n, dtype=np.float64)
    if kind == "descending":
        return -np.arange(n, dtype=np.float64)
    if kind == "signed_zeros":
        v = rng.integers(-1, 2, size=n).astype(np.float64)
        v[v == 0] = np.where(rng.random(int((v == 0).sum())) < 0.5, -0.0, 0.0)
        return v
    raise AssertionError(kind)


KINDS = ["uniform", "normal", "small_domain", "zipf_hi", "zipf_lo", "ascending", "descending", "signed_zeros"]


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("n,k", [(9_000, 100), (100_000, 1), (300_000, 1000), (1_000_000, 100),
                                 (1_000_000, 9000), (2_000_000, 100_000)])
def test_topk_random_vs_oracle(b200, kind, n, k):
    rng = np.random.default_rng(n * 31 + k + len(kind))
    keys = _gen(kind, n, rng)
    rows = rng.permutation(n).astype(np.uint32) if n % 2 else np.arange(n, dtype=np.uint32)
    got = b200.topk(KeyVector(keys, rows), k).payload.rows
    assert np.array_equal(got, oracle.topk(keys, rows, k))


def test_topk_k_at_least_n_is_full_descending_sort(b200):
    rng = np.random.default_rng(2)
    for n in (1, 2, 7, 8192, 8193, 20_000):
        keys = rng.integers(0, 50, size=n).astype(np.float64)
        rows = rng.permutation(n).astype(np.uint32)
        got = b200.topk(KeyVector(keys, rows), n + 5).payload.rows
        assert np.array_equal(got, oracle.topk(keys, rows, n + 5))


def test_topk_duplicate_rows_force_exact_fallback(b200):
    n = 3_000_000  # every (key, row) identical: the sampled threshold admits all n
    keys = np.full(n, 5.0)
    rows = np.full(n, 7, dtype=np.uint32)
    got = b200.topk(KeyVector(keys, rows), 50).payload.rows
    assert got.tolist() == [7] * 50


@pytest.mark.parametrize("env,fallback", [({}, 0), ({"GOLP_TOPK_CAP": "100"}, 1), ({"GOLP_TOPK_RANK_MAX": "64"}, 0),
                                          ({"GOLP_TOPK_FUSED": "0"}, 0)])
@pytest.mark.parametrize("kind", ["uniform", "small_domain", "zipf_hi"])
def test_topk_fused_path_and_in_kernel_fallbacks(b200, monkeypatch, env, fallback, kind):
    """C1-sized inputs run as one cooperative kernel; its in-kernel fallbacks
    (candidate buffer overflow -> direct select over the input, candidate list
    above the rank limit -> grid select over the candidates) must agree too."""
    from paper_2601_19911_b200 import _native

    for name, val in env.items():
        monkeypatch.setenv(name, val)
    rng = np.random.default_rng(77 + len(kind))
    n, k = 1_000_000, 100
    keys = _gen(kind, n, rng)
    rows = rng.permutation(n).astype(np.uint32)
    _native.check(_native.load().golp_set_profiling(1))
    try:
        got = b200.topk(KeyVector(keys, rows), k).payload.rows
        kt = _native.kernel_times()
    finally:
        _native.check(_native.load().golp_set_profiling(0))
    assert np.array_equal(got, oracle.topk(keys, rows, k))
    assert kt["topk_fallback"] == fallback
    assert kt["topk_candidates"] >= k


def test_topk_fused_identical_items(b200):
    n = 1_000_000  # identical (key, row) items: every item passes the threshold
    got = b200.topk(KeyVector(np.full(n, -2.5), np.full(n, 11, dtype=np.uint32)), 30).payload.rows
    assert got.tolist() == [11] * 30


def test_topk_empty_and_bad_k(b200):
    res = b200.topk(KeyVector(np.empty(0), np.empty(0, dtype=np.uint32)), 100)
    assert len(res.payload.rows) == 0 and res.ledger.h2d_bytes == 0
    with pytest.raises(ValueError):
        b200.topk(KeyVector(np.ones(3), np.arange(3)), 0)
    with pytest.raises(ValueError):
        b200.topk(KeyVector(np.ones(3), np.arange(3)), 1, mode=FULL_ROW)
    with pytest.raises(ValueError):
        b200.topk(KeyVector(np.ones(3), np.arange(3)), 1, mode="bogus")


def test_topk_full_row_same_answer_more_bytes(b200):
    rng = np.random.default_rng(12)
    kv = KeyVector(rng.standard_normal(10_000), np.arange(10_000))
    full = b200.topk(kv, 64, mode=FULL_ROW, payload_bytes=188)
    key = b200.topk(kv, 64)
    assert np.array_equal(full.payload.rows, key.payload.rows)
    assert full.ledger.h2d_bytes == 196 * 10_000 and key.ledger.h2d_bytes == 12 * 10_000
    led = key.ledger
    assert led.total == led.t_h2d + led.t_kernel + led.t_d2h + led.t_post
    assert led.t_h2d > 0 and led.t_kernel > 0


def test_topk_outputs_are_fresh_arrays(b200):
    kv = KeyVector(np.arange(1000, dtype=np.float64), np.arange(1000))
    a = b200.topk(kv, 10).payload.rows
    b = b200.topk(kv, 20).payload.rows
    assert a.tolist() == list(range(999, 989, -1))
    a[:] = 0  # caller may mutate; b must be unaffected
    assert b[0] == 999


def test_topk_resident_and_merge(cuda):
    import torch

    from paper_2601_19911_b200 import resident

    rng = np.random.default_rng(9)
    n, k = 5_000_000, 1000
    keys = rng.integers(0, 1000, size=n).astype(np.float64)
    rows = rng.permutation(n).astype(np.uint32)
    tk = torch.from_numpy(keys).to(cuda)
    tr = torch.from_numpy(rows.view(np.int32)).to(cuda)
    out, codes = resident.topk(tk, tr, k, want_codes=True)
    torch.cuda.synchronize()
    expect = oracle.topk(keys, rows, k)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), expect)
    # two halves -> local top-k -> merge == global top-k (the sharded algorithm)
    h = n // 2
    parts = [resident.topk(tk[s], tr[s], k, want_codes=True) for s in (slice(0, h), slice(h, n))]
    cat_rows = torch.cat([p[0] for p in parts])
    cat_codes = torch.cat([p[1] for p in parts])
    merged, _ = resident.merge(cat_codes, cat_rows, k)
    assert np.array_equal(merged.cpu().numpy().view(np.uint32), expect)
    assert _native.launch_count() > 0


def test_topk_large_uniform_known_properties(cuda):
    """1e8 uniform keys (800 MB): compare against the oracle's heap."""
    import torch

    from paper_2601_19911_b200 import resident

    n = 100_000_000
    rng = np.random.default_rng(7)
    keys = rng.integers(0, 2**53, size=n, dtype=np.int64).astype(np.float64)
    rows = np.arange(n, dtype=np.uint32)
    tk = torch.from_numpy(keys).to(cuda)
    tr = torch.from_numpy(rows.view(np.int32)).to(cuda)
    for k in (10, 1000, 100_000):
        out, _ = resident.topk(tk, tr, k)
        got = out.cpu().numpy().view(np.uint32)
        assert np.array_equal(got, oracle.topk(keys, rows, k)), k


@pytest.mark.parametrize("k,parts,domain", [(20_000, 4, 1 << 40), (50_000, 3, 5000), (8193, 2, 1 << 20)])
def test_topk_large_k_local_and_merge(cuda, k, parts, domain):
    """K above one shared-memory sort tile: the winners are sorted as 1024-item runs
    plus merge-path rounds, both in the local Top-K and in the cross-shard merge."""
    import torch

    from paper_2601_19911_b200 import resident

    rng = np.random.default_rng(k + parts)
    n = 3_000_000
    keys = rng.integers(0, domain, size=n).astype(np.float64)
    rows = rng.permutation(n).astype(np.uint32)
    tk = torch.from_numpy(keys).to(cuda)
    tr = torch.from_numpy(rows.view(np.int32)).to(cuda)
    expect = oracle.topk(keys, rows, k)
    out, _ = resident.topk(tk, tr, k, want_codes=True)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), expect)
    bounds = np.linspace(0, n, parts + 1).astype(int)
    res = [resident.topk(tk[a:b], tr[a:b], k, want_codes=True) for a, b in zip(bounds[:-1], bounds[1:])]
    merged, _ = resident.merge(torch.cat([r[1] for r in res]), torch.cat([r[0] for r in res]), k)
    assert np.array_equal(merged.cpu().numpy().view(np.uint32), expect)


@pytest.mark.parametrize("kind", ["uniform", "small_domain", "zipf_hi", "zipf_lo", "signed_zeros"])
@pytest.mark.parametrize("n,k,base", [(9_000, 100, 0), (1_000_000, 100, 0), (1_000_000, 9000, 12345),
                                      (3_000_000, 100_000, 0), (3_000_000, 1000, (1 << 32) - 3_000_000)])
def test_topk_positions_vs_oracle(cuda, kind, n, k, base):
    """Row ids given as positions (golp_topk_device_positions): no row column, the
    same answer as the explicit arange column (extract_keys's row ids)."""
    import torch

    from paper_2601_19911_b200 import resident

    rng = np.random.default_rng(n + k + len(kind))
    keys = _gen(kind, n, rng)
    rows = (np.arange(n, dtype=np.uint64) + base).astype(np.uint32)
    tk = torch.from_numpy(keys).to(cuda)
    out, codes = resident.topk(tk, base, k, want_codes=True)
    col, col_codes = resident.topk(tk, torch.from_numpy(rows.view(np.int32)).to(cuda), k, want_codes=True)
    torch.cuda.synchronize()
    expect = oracle.topk(keys, rows, k)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), expect)
    assert torch.equal(out, col) and torch.equal(codes, col_codes)


@pytest.mark.parametrize("env", [{"GOLP_TOPK_CAP": "100"}, {"GOLP_TOPK_RANK_MAX": "64"}, {"GOLP_TOPK_FUSED": "0"}])
def test_topk_positions_fallbacks(cuda, monkeypatch, env):
    import torch

    from paper_2601_19911_b200 import resident

    for name, v in env.items():
        monkeypatch.setenv(name, v)
    n, k, base = 1_000_000, 500, 77
    keys = _zipf(n, 5, True)
    rows = np.arange(base, base + n, dtype=np.uint32)
    out, _ = resident.topk(torch.from_numpy(keys).to(cuda), base, k)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), oracle.topk(keys, rows, k))


def test_topk_positions_sharded_merge_and_bounds(cuda):
    import torch

    from paper_2601_19911_b200 import resident

    n, k = 4_000_001, 1000
    keys = _zipf(n, 9, True)
    tk = torch.from_numpy(keys).to(cuda)
    h = n // 3
    parts = [resident.topk(tk[lo:hi], lo, k, want_codes=True) for lo, hi in ((0, h), (h, n))]
    merged, _ = resident.merge(torch.cat([p[1] for p in parts]), torch.cat([p[0] for p in parts]), k)
    expect = oracle.topk(keys, np.arange(n, dtype=np.uint32), k)
    assert np.array_equal(merged.cpu().numpy().view(np.uint32), expect)
    with pytest.raises(ValueError):
        resident.topk(tk, (1 << 32) - n + 1, k)  # row ids would pass 2^32 - 1
    lib = _native.load()
    assert lib.golp_topk_device_positions(tk.data_ptr(), n, (1 << 32) - n + 1, k, 0, 0, 0) != 0
