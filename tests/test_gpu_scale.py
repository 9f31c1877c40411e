"""Parity at the north-star sizes (BASELINE configs[2] and configs[3]).

C3: Top-K over N = 1e9 keys, K in {10, 1e3, 1e5}, uniform and Zipf-like keys
    (heavy ties on the largest key, "hi", and a heavy tail setting the threshold,
    "lo"), compared row for row with the oracle port of ProxyDevice.topk
    (pkg/src/golp/device.py:329-380, which equals host_topk, host.py:133-144).
C4: hash join, build 1e8 / probe 2e9 uniform keys in [0, 2e8), probed in ONE
    device call (radix-partitioned table, 2^30-probe spans, 64-bit pair
    offsets, ~1e9 pairs), compared span by span (2^28 probes) with the oracle's
    KeyHashTable probe (host.py:83-188) in reference pair order.

Inputs are generated on the device (torch, seeded) and copied to the host for
the oracle, so both sides see identical keys. The Zipf-like keys are an
inverse-transform sample r = floor(u^(-1/(a-1))), a = 1.2, clipped to 2^53 - 1
(numpy's exact zipf sampler needs minutes at 1e9); SURVEY 8(d)'s key maps are
applied: hi = (2^53 - 1) - r, lo = r.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

N_C3 = 1_000_000_000
KS = (10, 1_000, 100_000)
THREADS = os.cpu_count() or 1


def _scrambled_rows(torch, n, dev):
    """Distinct, non-monotone u32 row ids: i * 0x9E3779B1 mod 2^32 (a bijection)."""
    i = torch.arange(n, dtype=torch.int64, device=dev)
    return ((i * 0x9E3779B1) & 0xFFFFFFFF).to(torch.int32)


def _keys(torch, dist, n, dev):
    g = torch.Generator(device=dev).manual_seed({"uniform": 7, "zipf_hi": 11, "zipf_lo": 11}[dist])
    if dist == "uniform":  # random_keys (store.py:165-171): integers in [0, 2^53) as f8
        return torch.randint(0, 2**53, (n,), dtype=torch.int64, device=dev, generator=g).to(torch.float64)
    u = 1.0 - torch.rand(n, dtype=torch.float64, device=dev, generator=g)  # (0, 1]
    r = torch.floor(torch.clamp(u.pow_(-5.0), max=2.0**53 - 1))
    return (2.0**53 - 1) - r if dist == "zipf_hi" else r


@pytest.fixture(scope="module", params=["uniform", "zipf_hi", "zipf_lo"])
def c3_data(request, cuda):
    import torch

    dist = request.param
    keys = _keys(torch, dist, N_C3, cuda)
    rows = _scrambled_rows(torch, N_C3, cuda) if dist == "zipf_hi" else \
        torch.arange(N_C3, dtype=torch.int32, device=cuda)
    yield dist, keys, rows, keys.cpu().numpy(), rows.cpu().numpy().view(np.uint32)
    del keys, rows
    torch.cuda.empty_cache()


@pytest.mark.parametrize("k", KS)
def test_c3_topk_1e9_matches_oracle(c3_data, k):
    from paper_2601_19911_b200 import resident

    dist, keys, rows, hk, hr = c3_data
    got, _ = resident.topk(keys, rows, k)
    want = oracle.proxy_topk(hk, hr, k, THREADS)
    np.testing.assert_array_equal(got.cpu().numpy().view(np.uint32), want, err_msg=f"C3 {dist} k={k}")


def test_c3_topk_1e9_end_to_end_from_host(c3_data, b200):
    """The public device-protocol call from host numpy columns (chunked upload)."""
    from paper_2601_19911_b200 import KeyVector

    dist, _, _, hk, hr = c3_data
    if dist != "uniform":
        pytest.skip("one end-to-end case is enough; the kernels are covered above")
    res = b200.topk(KeyVector(hk, hr), 1_000)
    np.testing.assert_array_equal(res.payload.rows, oracle.proxy_topk(hk, hr, 1_000, THREADS))
    assert res.ledger.h2d_bytes == 12 * N_C3


NB_C4, NP_C4 = 100_000_000, 2_000_000_000
SPAN = 1 << 28


def test_c4_join_1e8_by_2e9_matches_oracle_span_by_span(cuda):
    import torch

    from paper_2601_19911_b200 import _native, resident

    g = torch.Generator(device=cuda).manual_seed(1)
    dom = 2 * NB_C4
    bk = torch.randint(0, dom, (NB_C4,), dtype=torch.int64, device=cuda, generator=g).to(torch.float64)
    br = torch.arange(NB_C4, dtype=torch.int32, device=cuda)
    pk = torch.empty(NP_C4, dtype=torch.float64, device=cuda)
    for s in range(0, NP_C4, SPAN):  # chunked: no 16 GB int64 temporary
        e = min(s + SPAN, NP_C4)
        pk[s:e] = torch.randint(0, dom, (e - s,), dtype=torch.int64, device=cuda, generator=g).to(torch.float64)
    pr = torch.arange(NP_C4, dtype=torch.int32, device=cuda)
    cap = NP_C4 // 2 + NP_C4 // 8
    op = torch.empty(cap, dtype=torch.int32, device=cuda)
    ob = torch.empty(cap, dtype=torch.int32, device=cuda)
    resident.set_profiling(True)
    resident.join_build(bk, br)
    m = resident.join_probe(pk, pr, op, ob)
    kt = _native.kernel_times()
    resident.set_profiling(False)
    assert kt["join_slices"] > 1, "C4 must take the radix-partitioned path"
    assert m > 2**32 // 8  # ~1e9 pairs: offsets beyond 2^31 entries of each array are exercised

    table = oracle.Table(bk.cpu().numpy(), br.cpu().numpy().view(np.uint32))
    del bk, br
    cum = 0
    for s in range(0, NP_C4, SPAN):
        e = min(s + SPAN, NP_C4)
        hk = pk[s:e].cpu().numpy()
        hr = np.arange(s, e, dtype=np.uint32)
        wp, wb = table.probe(hk, hr, workers=THREADS)
        n = len(wp)
        gp = op[cum:cum + n].cpu().numpy().view(np.uint32)
        gb = ob[cum:cum + n].cpu().numpy().view(np.uint32)
        np.testing.assert_array_equal(gp, wp, err_msg=f"probe rows, span at {s}")
        np.testing.assert_array_equal(gb, wb, err_msg=f"build rows, span at {s}")
        cum += n
    assert cum == m
