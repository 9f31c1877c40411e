"""The drop-in claim, checked against the real reference package.

The UNMODIFIED reference `golp` (installed into baseline/_ref by
baseline/install_reference.sh, with its independent test oracles
pkg/tests/oracles.py) runs its own code paths with `B200Device` plugged in as
the device: golp's KeyVectors, tables, gate (execute_path / execute_gated,
pkg/src/golp/gate.py:167-233) and harness (run_strategy_comparison,
run_payload_comparison, pkg/src/golp/harness.py:290-415) call the B200 backend
through the duck-typed device protocol and read its results and ledgers. The
checks restate the reference's own tests with the device substituted:
criterion 1 (pkg/tests/test_acceptance.py:74-105), the proxy multi-chunk and
ledger tests (pkg/tests/test_device.py:169-238) and the _LyingDevice negative
case (pkg/tests/test_harness.py:218-229).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
if not (REF / "golp").exists():
    pytest.skip("the reference package is not installed (run baseline/install_reference.sh)",
                allow_module_level=True)
sys.path.insert(0, str(REF))

import golp  # noqa: E402
from golp.device import FULL_ROW, KEY_ONLY, OP_PROBE, OP_TOPK, ModeledDevice, device_topk  # noqa: E402
from golp.errors import StrategyMismatchError  # noqa: E402
from golp.gate import DEVICE, HOST, GateConfig, execute_gated, execute_path  # noqa: E402
from golp.harness import WorkloadSpec, run_payload_comparison, run_strategy_comparison  # noqa: E402
from golp.host import host_hash_build, host_hash_probe, host_topk  # noqa: E402
from golp.store import KeyVector, generate_table, random_key_vector  # noqa: E402
from golp_ref_tests.oracles import oracle_join_outer, oracle_topk_rows  # noqa: E402


def _chunked_join_oracle(bk, br, pk, pr, max_cells=4_000_000):  # test_acceptance.py:60-66
    step = max(1, max_cells // max(1, len(bk)))
    out = []
    for lo in range(0, len(pk), step):
        out.extend(oracle_join_outer(bk, br, pk[lo:lo + step], pr[lo:lo + step]))
    return out


def test_golp_is_the_unmodified_reference():
    assert Path(golp.__file__).resolve().is_relative_to(REF.resolve())


def test_criterion_01_with_the_b200_device(b200):
    """Crit 1's 200 Top-K + 200 probe instances (same seed and generator) on the
    B200, against the reference's brute-force oracles, with golp KeyVectors."""
    rng = np.random.default_rng(20260816)
    for i in range(200):
        n = int(10 ** rng.uniform(1, 5))
        k = int(rng.choice([1, 10, 100, max(1, n)]))
        keys = rng.integers(0, max(2, n // 8), size=n).astype(np.float64) if i % 3 == 0 else rng.standard_normal(n)
        kv = KeyVector(keys=keys, rows=rng.permutation(n).astype(np.uint32))
        expect = oracle_topk_rows(keys.tolist(), kv.rows.tolist(), k)
        assert list(b200.topk(kv, k).payload.rows) == expect, f"b200 topk diverged (n={n}, k={k})"
    for i in range(200):
        nb = int(10 ** rng.uniform(1, 4))
        npr = int(10 ** rng.uniform(1, 4))
        domain = max(4, (nb + npr) // 3)
        bk = rng.integers(0, domain, size=nb).astype(np.float64)
        pk = rng.integers(0, domain, size=npr).astype(np.float64)
        build = KeyVector(keys=bk, rows=rng.permutation(nb).astype(np.uint32))
        probe = KeyVector(keys=pk, rows=rng.permutation(npr).astype(np.uint32))
        expect = _chunked_join_oracle(bk, build.rows, pk, probe.rows)
        assert b200.probe(build, probe).payload.matches == expect, f"b200 probe diverged (nb={nb}, np={npr})"


def _small_domain_keys(n, seed, domain=50):  # test_device.py's helper, restated
    rng = np.random.default_rng(seed)
    return KeyVector(keys=rng.integers(0, domain, size=n).astype(np.float64), rows=np.arange(n, dtype=np.uint32))


def test_device_protocol_tests_with_the_b200_device(b200):
    """test_device.py:169-238 with ProxyDevice replaced by B200Device."""
    keys = _small_domain_keys(20_000, 9)
    res = b200.topk(keys, 100)
    assert res.backend == "b200"
    assert np.array_equal(res.payload.rows, host_topk(keys, 100).rows)
    keys = random_key_vector(10_000, 12)
    full = b200.topk(keys, 64, mode=FULL_ROW, payload_bytes=188)
    key = b200.topk(keys, 64)
    assert np.array_equal(full.payload.rows, key.payload.rows)
    assert full.ledger.h2d_bytes == 196 * 10_000 and key.ledger.h2d_bytes == 12 * 10_000
    build, probe = _small_domain_keys(5_000, 4, domain=512), _small_domain_keys(20_000, 5, domain=512)
    res = b200.probe(build, probe)
    expect = host_hash_probe(host_hash_build(build), probe)
    assert res.payload.matches == expect.matches and res.payload.probe_count == expect.probe_count
    keys = random_key_vector(8_192, 8)
    got, modeled = b200.topk(keys, 100), device_topk(keys, 100)
    assert got.ledger.h2d_bytes == modeled.ledger.h2d_bytes and got.ledger.d2h_bytes == modeled.ledger.d2h_bytes
    led = b200.topk(random_key_vector(4_096, 2), 10).ledger
    assert led.total == led.t_h2d + led.t_kernel + led.t_d2h + led.t_post
    assert led.t_h2d > 0.0 and led.t_kernel > 0.0


def test_golp_gate_runs_queries_on_the_b200(b200):
    """golp's execute_path / execute_gated with the B200 backend: same answers as
    golp's own host path, wall-clock latencies, probes unmaterialized (as golp)."""
    t = generate_table(300_000, 16, seed=5)
    dev_res, dev_lat = execute_path(t, OP_TOPK, 1000, GateConfig(), b200, DEVICE)
    host_res, _ = execute_path(t, OP_TOPK, 1000, GateConfig(), b200, HOST)
    assert np.array_equal(dev_res.row_ids, host_res.row_ids) and np.array_equal(dev_res.payloads, host_res.payloads)
    assert dev_lat > 0
    big = generate_table(3_000_000, 4, seed=2)
    res, decision, lat = execute_gated(big, OP_TOPK, 100, GateConfig(), device=b200)
    assert decision.path == DEVICE and len(res.row_ids) == 100 and lat > 0
    assert np.array_equal(res.row_ids, host_topk(KeyVector(big.key_column, np.arange(big.row_count,
                                                                                      dtype=np.uint32)), 100).rows)
    bt, pt = generate_table(2_000, 8, seed=6), generate_table(30_000, 8, seed=7)
    p_dev, _ = execute_path((bt, pt), OP_PROBE, 1, GateConfig(), b200, DEVICE)
    p_host, _ = execute_path((bt, pt), OP_PROBE, 1, GateConfig(), b200, HOST)
    assert p_dev.matches == p_host.matches and p_dev.probe_count == p_host.probe_count


def test_golp_strategy_and_payload_comparisons_on_the_b200(b200):
    """golp's harness cross-checks every strategy's answers per n (a mismatch
    raises) and reads the B200 ledgers for the key-only vs full-row rows."""
    spec = WorkloadSpec(n_grid=(1_000, 20_000, 100_000), repeats=3, payload_bytes=16, k=100)
    host, device, gated = run_strategy_comparison(spec, GateConfig(), device=b200)
    assert host.offload_rate == 0.0 and device.offload_rate == 1.0
    mixed = WorkloadSpec(n_grid=(10_000, 200_000), repeats=20, mix=(0.8, 0.2), seed=3, payload_bytes=16)
    run_strategy_comparison(mixed, GateConfig(), device=b200)
    spec = WorkloadSpec(n_grid=(100_000, 1_000_000), repeats=1, k=100, payload_bytes=188)
    cmp_b200 = run_payload_comparison(spec, device=b200)
    cmp_model = run_payload_comparison(spec, device=ModeledDevice())
    bytes_b200 = [(r.n, r.mode, r.bytes) for r in cmp_b200.payload_rows]
    assert bytes_b200 == [(r.n, r.mode, r.bytes) for r in cmp_model.payload_rows]
    for r in cmp_b200.e2e_rows:
        if r.mode == KEY_ONLY:
            assert r.speedup_vs_full_row > 1.0  # key-only beats shipping 196-byte rows


class _LyingB200:
    """B200Device with correct ledgers but the wrong rows (test_harness.py:218-224)."""

    name = "b200"

    def __init__(self, dev):
        self._dev = dev

    def topk(self, keys, k, mode=KEY_ONLY, payload_bytes=None):
        call = self._dev.topk(keys, k, mode=mode, payload_bytes=payload_bytes)
        call.payload.rows[:] = call.payload.rows[::-1]
        return call


def test_divergent_b200_answers_abort_golps_comparison(b200):
    spec = WorkloadSpec(n_grid=(1_000, 20_000), repeats=2, payload_bytes=16, k=50)
    with pytest.raises(StrategyMismatchError):
        run_strategy_comparison(spec, GateConfig(), device=_LyingB200(b200))
