"""Dense row-id elision on the host-buffer path: a row-id column that is a
dense run (rows[i] == rows[0] + i mod 2^32, what extract_keys makes,
pkg/src/golp/store.py:178-181) is verified on the host and regenerated on the
device instead of copied. Results must not change for any column -- dense,
offset, wrapping past 2^32, dense except one entry, or dense except one
staging chunk -- and the bytes actually moved must say which columns crossed
PCIe."""

import numpy as np
import pytest

from oracle import oracle
from paper_2601_19911_b200 import B200Device, KeyVector, _native

pytestmark = pytest.mark.gpu

CHUNK = 2 << 20  # entries per staging chunk (16 MB of keys, the library default)


def _rows(kind, n, rng):
    r = np.arange(n, dtype=np.uint64)
    if kind == "arange":
        pass
    elif kind == "offset":
        r = r + 1000
    elif kind == "wrap":  # crosses 2^32 - 1 -> 0 halfway
        r = r + (1 << 32) - n // 2
    elif kind == "high":  # ends at 2^32 - 2, the largest row id a build table can hold
        r = r + (1 << 32) - 1 - n
    elif kind == "swap_middle":
        m = n // 2 + 3
        r[[m, m + 1]] = r[[m + 1, m]]
    elif kind == "swap_last":
        r[[n - 2, n - 1]] = r[[n - 1, n - 2]]
    elif kind == "one_chunk_permuted":
        lo, hi = CHUNK, min(n, 2 * CHUNK)
        r[lo:hi] = lo + rng.permutation(hi - lo)
    elif kind == "descending":
        r = r[::-1].copy()
    return (r % (1 << 32)).astype(np.uint32)


def _dense(r):
    return len(r) < 2 or bool(np.all(r == (r[0] + np.arange(len(r), dtype=np.uint64)) % (1 << 32)))


def _elided(rows, chunked):
    """Bytes of row ids the library should not copy: 4 per entry of every
    upload unit (the whole column, or each staging chunk) that is a dense run."""
    units = [rows[i:i + CHUNK] for i in range(0, len(rows), CHUNK)] if chunked else [rows]
    return sum(4 * len(u) for u in units if _dense(u))


KINDS = ["arange", "offset", "wrap", "high", "swap_middle", "swap_last", "one_chunk_permuted", "descending"]
DENSE = {"arange", "offset", "wrap", "high"}
# The reference's hash table reserves row 0xFFFFFFFF as its empty-slot marker
# ("rowids cap at 2**32 - 2", pkg/src/golp/host.py:17), so join inputs never wrap.
PROBE_KINDS = [k for k in KINDS if k != "wrap"]


@pytest.fixture(scope="module")
def copied():
    dev = B200Device(dense_rows=False)
    yield dev
    dev.close()


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("n,k,domain", [(1_000_000, 100, 1 << 53), (5_000_000, 1000, 1 << 53),
                                        (5_000_000, 100_000, 50)])
def test_topk_dense_rows_same_answer(b200, copied, kind, n, k, domain):
    rng = np.random.default_rng(n + k + domain)
    keys = rng.integers(0, domain, size=n).astype(np.float64)
    rows = _rows(kind, n, rng)
    got = b200.topk(KeyVector(keys, rows), k).payload.rows
    h2d, d2h = _native.last_transfer()
    ref = copied.topk(KeyVector(keys, rows), k).payload.rows
    h2d_copied, _ = _native.last_transfer()
    assert np.array_equal(got, ref)
    if domain < 1000 or n <= 1_000_000:  # heavy ties / C1 size: also against the oracle
        assert np.array_equal(got, oracle.topk(keys, rows, k))
    assert d2h == 4 * min(k, n)
    assert h2d_copied - h2d == _elided(rows, chunked=n > CHUNK)
    if kind in DENSE:
        assert h2d_copied - h2d == 4 * n


@pytest.mark.parametrize("kind", PROBE_KINDS)
def test_probe_dense_rows_same_answer(b200, copied, kind):
    nb, np_, domain = 1_000_000, 5_000_000, 2_000_000
    rng = np.random.default_rng(7)
    bk = rng.integers(0, domain, size=nb).astype(np.float64)
    pk = rng.integers(0, domain, size=np_).astype(np.float64)
    br, pr = _rows(kind, nb, rng), _rows(kind, np_, rng)
    got = b200.probe(KeyVector(bk, br), KeyVector(pk, pr)).payload
    h2d, d2h = _native.last_transfer()
    ep, eb = oracle.join(bk, br, pk, pr)
    assert np.array_equal(got.probe_rows, ep) and np.array_equal(got.build_rows, eb)
    assert d2h == 8 * len(ep)
    ref = copied.probe(KeyVector(bk, br), KeyVector(pk, pr)).payload
    assert np.array_equal(ref.probe_rows, ep) and np.array_equal(ref.build_rows, eb)
    h2d_copied, _ = _native.last_transfer()
    assert h2d_copied == 12 * (nb + np_)
    assert h2d_copied - h2d == _elided(br, chunked=False) + _elided(pr, chunked=True)
    if kind in DENSE:
        assert h2d == 8 * (nb + np_)


@pytest.mark.parametrize("n", [1, 2, 3, 1000])
def test_tiny_dense_columns(b200, n):
    keys = np.arange(n, dtype=np.float64)[::-1].copy()
    rows = np.arange(n, dtype=np.uint32) + 7
    assert b200.topk(KeyVector(keys, rows), 2).payload.rows.tolist() == rows[: min(2, n)].tolist()
    res = b200.probe(KeyVector(keys, rows), KeyVector(keys[::-1].copy(), rows))
    assert res.payload.match_count == n
    ep, eb = oracle.join(keys, rows, keys[::-1].copy(), rows)
    assert np.array_equal(res.payload.probe_rows, ep) and np.array_equal(res.payload.build_rows, eb)


def test_full_sort_dense_rows_same_answer(b200, copied):
    rng = np.random.default_rng(5)
    n = 3_000_000
    keys = rng.integers(0, 1000, size=n).astype(np.float64)
    for kind in ("arange", "wrap", "swap_middle"):
        rows = _rows(kind, n, rng)
        got = b200.full_sort(KeyVector(keys, rows)).payload
        ref = copied.full_sort(KeyVector(keys, rows)).payload
        assert np.array_equal(got, ref)
        assert np.array_equal(got, rows[np.lexsort((rows, keys))])


@pytest.mark.parametrize("bkind,pkind", [("arange", "permuted"), ("permuted", "arange"), ("arange", "arange")])
def test_probe_mixed_density_and_full_row(b200, bkind, pkind):
    """Dense and copied row columns on either side, key-only and full-row mode
    (the full-row payload stream shares the copy queue with the key chunks)."""
    from paper_2601_19911_b200 import FULL_ROW

    rng = np.random.default_rng(41)
    nb, np_ = 300_000, 4_500_000
    bk = rng.integers(0, 2 * nb, size=nb).astype(np.float64)
    pk = rng.integers(0, 2 * nb, size=np_).astype(np.float64)
    mk = lambda kind, n: (np.arange(n, dtype=np.uint32) if kind == "arange"  # noqa: E731
                          else rng.permutation(n).astype(np.uint32))
    br, pr = mk(bkind, nb), mk(pkind, np_)
    ep, eb = oracle.join(bk, br, pk, pr)
    for mode, pb in (("key_only", None), (FULL_ROW, 20)):
        res = b200.probe(KeyVector(bk, br), KeyVector(pk, pr), mode=mode, payload_bytes=pb)
        assert np.array_equal(res.payload.probe_rows, ep) and np.array_equal(res.payload.build_rows, eb)


@pytest.mark.parametrize("kind", ["arange", "one_chunk_permuted"])
def test_topk_full_row_chunked_dense_rows(b200, kind):
    from paper_2601_19911_b200 import FULL_ROW

    rng = np.random.default_rng(43)
    n = 5_000_000
    keys = rng.integers(0, 1 << 53, size=n).astype(np.float64)
    rows = _rows(kind, n, rng)
    got = b200.topk(KeyVector(keys, rows), 500, mode=FULL_ROW, payload_bytes=12).payload.rows
    assert np.array_equal(got, oracle.topk(keys, rows, 500))


@pytest.mark.parametrize("n", [CHUNK - 1, CHUNK, CHUNK + 1, 2 * CHUNK + 1, 2 * CHUNK + 63])
def test_chunk_boundaries_dense_rows(b200, n):
    """Inputs one entry either side of the staging-chunk size: single-entry tail
    chunks are dense runs by definition and must be filled, not skipped."""
    rng = np.random.default_rng(n)
    keys = rng.integers(0, 1 << 53, size=n).astype(np.float64)
    rows = np.arange(n, dtype=np.uint32) + 5
    keys[-1] = float(1 << 53)  # the last entry is the maximum: it must come back first
    got = b200.topk(KeyVector(keys, rows), 50).payload.rows
    assert got[0] == rows[-1]
    assert np.array_equal(got, oracle.topk(keys, rows, 50))
    bk = rng.integers(0, 1000, size=3000).astype(np.float64)
    pk = rng.integers(0, 1000, size=n).astype(np.float64)
    pr = rows
    res = b200.probe(KeyVector(bk, np.arange(3000, dtype=np.uint32)), KeyVector(pk, pr)).payload
    ep, eb = oracle.join(bk, np.arange(3000, dtype=np.uint32), pk, pr)
    assert np.array_equal(res.probe_rows, ep) and np.array_equal(res.build_rows, eb)
