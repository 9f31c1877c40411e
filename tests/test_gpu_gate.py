"""Risky Gate with the B200 backend: calibrated profile from real ledgers,
strategy comparison (answers cross-checked between the host engine and the
device on every query), gated execution of both ops."""

import numpy as np
import pytest

from paper_2601_19911_b200 import DEVICE, HOST, OP_PROBE, OP_TOPK, GateConfig, execute_gated, execute_path, generate_table
from paper_2601_19911_b200.harness import (
    WorkloadSpec,
    calibrate_device_profile,
    compute_stats,
    run_strategy_comparison,
)

pytestmark = pytest.mark.gpu


def test_b200_profile_calibrates_and_strategies_agree(b200):
    prof = calibrate_device_profile(b200, ns=(50_000, 200_000, 800_000, 2_000_000), repeats=2)
    assert prof.h2d_bandwidth > 1e9 and prof.launch_overhead > 0
    cfg = GateConfig(profile=prof, min_n_guard=20_000)
    spec = WorkloadSpec(n_grid=(10_000, 100_000, 1_000_000), repeats=3, payload_bytes=16, k=100)
    host, device, gated = run_strategy_comparison(spec, cfg, device=b200)  # raises on any mismatch
    assert device.offload_rate == 1.0 and host.offload_rate == 0.0
    for run in (host, device, gated):
        s = compute_stats(run.all_samples())
        assert s.p99 >= s.p95 >= s.median > 0


def test_device_and_host_paths_return_identical_results(b200):
    t = generate_table(300_000, 8, seed=5)
    cfg = GateConfig()
    r_dev, _ = execute_path(t, OP_TOPK, 1000, cfg, b200, DEVICE)
    r_host, _ = execute_path(t, OP_TOPK, 1000, cfg, b200, HOST)
    assert np.array_equal(r_dev.row_ids, r_host.row_ids)
    assert np.array_equal(r_dev.payloads, r_host.payloads)
    bt = generate_table(50_000, 8, seed=6)
    p_dev, _ = execute_path((bt, t), OP_PROBE, 1, cfg, b200, DEVICE)
    p_host, _ = execute_path((bt, t), OP_PROBE, 1, cfg, b200, HOST)
    assert p_dev.matches == p_host.matches


def test_execute_gated_offloads_large_queries(b200):
    t = generate_table(3_000_000, 4, seed=2)
    res, d, lat = execute_gated(t, OP_TOPK, 100, GateConfig(), device=b200)
    assert d.path == DEVICE and len(res) == 100 and lat > 0


def test_scaling_baseline_with_b200_rows(b200):
    from paper_2601_19911_b200.harness import WorkloadSpec, run_scaling_baseline

    rows = run_scaling_baseline(WorkloadSpec(n_grid=(10_000, 200_000), k=100, repeats=3), backend="host",
                                device=b200)
    ops = {(r.n, r.op) for r in rows}
    assert (200_000, "full_sort@b200") in ops and (200_000, "topk@b200") in ops
    assert all(r.median_s > 0 for r in rows)


def _join_tables(nb, np_, payload_bytes, seed):
    """Build / probe ColumnTables with C2-style join keys (uniform integers in [0, 2*nb) as f8)."""
    from paper_2601_19911_b200.store import ColumnTable

    rng = np.random.Generator(np.random.PCG64(seed))
    bk = rng.integers(0, 2 * nb, size=nb).astype(np.float64)
    pk = rng.integers(0, 2 * nb, size=np_).astype(np.float64)
    bp = (np.arange(nb * payload_bytes, dtype=np.uint64) * 2654435761 % 251).astype(np.uint8).reshape(nb, payload_bytes)
    pp = (np.arange(np_ * payload_bytes, dtype=np.uint64) * 40503 % 241).astype(np.uint8).reshape(np_, payload_bytes)
    return ColumnTable(bk, bp, seed), ColumnTable(pk, pp, seed + 1)


@pytest.mark.parametrize("path", [DEVICE, HOST])
def test_join_late_materialization_on_the_query_path_c2(b200, path):
    """execute_path with materialize_joins: pairs in reference order, then both
    sides' keys + payloads gathered in pair order (store.materialize semantics,
    pkg/src/golp/store.py:184-201), at the C2 shape (build 1e6 / probe 1e7)."""
    from oracle import oracle

    nb, np_ = (1_000_000, 10_000_000) if path == DEVICE else (100_000, 1_000_000)
    bt, pt = _join_tables(nb, np_, 16, seed=1)
    cfg = GateConfig(materialize_joins=True)
    res, lat = execute_path((bt, pt), OP_PROBE, 1, cfg, b200, path)
    ep, eb = oracle.join(bt.key_column, bt.positions, pt.key_column, pt.positions)
    assert len(res) == len(ep) and lat > 0
    assert np.array_equal(res.probe.row_ids, ep) and np.array_equal(res.build.row_ids, eb)
    assert np.array_equal(res.probe.keys, pt.key_column[ep]) and np.array_equal(res.build.keys, bt.key_column[eb])
    assert np.array_equal(res.probe.keys, res.build.keys)  # an equi-join
    assert np.array_equal(res.probe.payloads, pt.payload_column[ep])
    assert np.array_equal(res.build.payloads, bt.payload_column[eb])
    assert GateConfig.from_json_dict(cfg.to_json_dict()) == cfg
    assert "materialize_joins" not in GateConfig().to_json_dict()


def test_calibrated_profile_kernel_terms_are_device_timed(b200):
    """C_gpu's kernel term comes from CUDA-event kernel times (not the wall-clock
    tail after the last upload), so no kernel rate sits at the fit's clamp."""
    prof = calibrate_device_profile(b200, ns=(250_000, 1_000_000, 4_000_000, 16_000_000),
                                    probe_ns=(500_000, 2_000_000, 8_000_000), repeats=3)
    assert prof.kernel_rate_topk > 1e-12 and prof.kernel_rate_probe > 1e-12
    # device rates: Top-K well above 10 Gkeys/s, build+probe above 1 Gkeys/s
    assert prof.kernel_rate_topk < 1e-10 and prof.kernel_rate_probe < 1e-9
    assert 20e9 < prof.h2d_bandwidth < 200e9  # per reference byte (12 B/entry accounted, 8 moved)


def test_criterion_07_stream_on_b200(b200):
    """Reference acceptance criterion 7 (pkg/tests/test_acceptance.py:252-270) on
    real hardware: the 500-query 80/20 stream (n in {1e4, 1e6}, seed 3, 188-B
    payloads) under host_only / device_always / gated, three runs. The gate
    sends 1e4 to the host and 1e6 to the device, so it beats both fixed
    strategies at P50 and host_only everywhere; its P95/P99 are the same device
    calls as device_always's tail: standalone runs put them 0.3-7% above
    device_always's, inside a long test session up to ~11% (host-side state,
    not a different path, separates them: DESIGN.md §7), so the bound here is
    25%. The gate's 1e4 queries take host_only's own path, so their P50s agree up
    to noise (standalone the gate's is lower; inside the suite the two have
    measured within 3% either way): 10% bound there. The reference asserts no P50."""
    spec = WorkloadSpec(n_grid=(10_000, 1_000_000), repeats=250, mix=(0.8, 0.2), seed=3)
    assert len(spec.n_grid) * spec.repeats == 500
    tables = {}
    for _ in range(3):
        host, device, gated = run_strategy_comparison(spec, GateConfig(), device=b200, tables=tables)
        h, d, g = (compute_stats(r.all_samples()) for r in (host, device, gated))
        assert 0.1 < gated.offload_rate < 0.3
        assert g.median <= 1.1 * h.median and g.median < d.median
        assert g.p95 <= h.p95 and g.p99 <= h.p99
        assert g.p95 <= 1.25 * d.p95 and g.p99 <= 1.25 * d.p99


def test_cli_bench_on_the_b200(tmp_path, b200):
    """`cli bench --backend b200`: calibrated gate, B200 rows in every output."""
    import json

    from paper_2601_19911_b200 import cli

    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"workload": {"n_grid": [10_000, 200_000, 1_000_000], "repeats": 3,
                                            "payload_bytes": 16}}))
    assert cli.main(["bench", "--config", str(cfg), "--backend", "b200", "--out", str(tmp_path / "out")]) == 0
    summary = json.loads((tmp_path / "out" / "summary.json").read_text())
    assert summary["backend"] == "b200" and summary["gate"]["profile"]["kernel_rate_topk"] > 1e-12
    assert "topk@b200" in (tmp_path / "out" / "scaling.csv").read_text()
