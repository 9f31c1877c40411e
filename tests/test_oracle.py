"""Pins the oracle (oracle/oracle.c) to the reference's own outputs.

The golden vectors were produced by running /root/reference's golp package
(tests/golden/make_golden.py); nothing here re-derives them.
"""

import numpy as np
import pytest

from golden_io import cases, npz
from oracle import oracle


@pytest.mark.parametrize("case", cases("topk"), ids=lambda c: f"{c['tag']}-n{len(c['keys'])}-k{c['k']}")
def test_oracle_topk_matches_reference(case):
    got = oracle.topk(case["keys"], case["rows"], int(case["k"]))
    assert got.tolist() == case["expect"].tolist()


@pytest.mark.parametrize("case", cases("probe"), ids=lambda c: f"{c['tag']}-{len(c['bkeys'])}x{len(c['pkeys'])}")
def test_oracle_join_matches_reference(case):
    p, b = oracle.join(case["bkeys"], case["brows"], case["pkeys"], case["prows"])
    assert p.tolist() == case["exp_p"].tolist()
    assert b.tolist() == case["exp_b"].tolist()


def test_oracle_table_layout_and_mix64_match_reference():
    z = npz("table")
    t = oracle.Table(z["keys"], z["rows"])
    assert t.capacity == int(z["capacity"])
    assert np.array_equal(t.slot_bits, z["slot_bits"])
    assert np.array_equal(t.slot_rows, z["slot_rows"])
    assert [oracle.mix64(int(v)) for v in z["mix_in"].tolist()] == z["mix_out"].tolist()


def test_oracle_topk_large_known_answer():
    from paper_2601_19911_b200.store import random_key_vector

    z = npz("topk_large")
    kv = random_key_vector(int(z["n"]), int(z["seed"]))
    assert np.array_equal(kv.keys[:16], z["key_head"])  # generator parity with the reference
    assert kv.keys.sum() == z["key_sum"]
    assert oracle.topk(kv.keys, kv.rows, int(z["k"])).tolist() == z["expect"].tolist()


@pytest.mark.parametrize("workers", [1, 3, 8])
def test_oracle_proxy_ports_agree_with_oracle(workers):
    rng = np.random.default_rng(workers)
    keys = rng.integers(0, 300, size=50_000).astype(np.float64)
    rows = rng.permutation(50_000).astype(np.uint32)
    for k in (1, 100, 4096):
        assert np.array_equal(oracle.proxy_topk(keys, rows, k, workers), oracle.topk(keys, rows, k))
    t = oracle.Table(keys[:5000], rows[:5000])
    p1, b1 = t.probe(keys, rows, workers=1)
    pw, bw = t.probe(keys, rows, workers=workers)
    assert np.array_equal(p1, pw) and np.array_equal(b1, bw)


@pytest.mark.parametrize("case", cases("full_sort"), ids=lambda c: f"{c['tag']}-n{len(c['keys'])}")
def test_oracle_full_sort_matches_reference(case):
    assert oracle.full_sort(case["keys"], case["rows"]).tolist() == case["expect"].tolist()
