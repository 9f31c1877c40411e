"""Gate / cost model / calibration / statistics against the reference's own
numbers (tests/golden/gate.json, produced by running golp), plus the
reference's behavioural gate tests restated on this package."""

import math

import numpy as np
import pytest

from golden_io import gate_golden
from paper_2601_19911_b200 import (
    DEFAULT_CPU_MODEL,
    DEFAULT_MODELED_PROFILE,
    DEVICE,
    FULL_ROW,
    HOST,
    KEY_ONLY,
    OP_PROBE,
    OP_TOPK,
    CalibrationError,
    CpuCostModel,
    DeviceProfile,
    GateConfig,
    ModeledDevice,
    StrategyMismatchError,
    TransferLedger,
    calibrate_cpu_model,
    calibrate_profile,
    decide,
    estimate_cpu_cost,
    estimate_device_cost,
    execute_gated,
    generate_table,
    transfer_entry_bytes,
    with_margin,
)
from paper_2601_19911_b200.harness import (
    WorkloadSpec,
    compute_stats,
    run_payload_comparison,
    run_strategy_comparison,
)

G = gate_golden()
CFGS = {
    "default": GateConfig(),
    "margin5ms": GateConfig(margin_s=5e-3),
    "guard20k": GateConfig(min_n_guard=20_000),
    "full_row": GateConfig(mode=FULL_ROW),
}


def test_decide_matches_reference_on_every_grid_point():
    assert len(G["decide"]) > 300
    for name, op, n, k, build_n, path, c_cpu, c_gpu, gain, guard in G["decide"]:
        cfg = CFGS[name]
        pb = 188 if cfg.mode == FULL_ROW else None
        d = decide(cfg, op, n, k, pb, build_n)
        assert (d.path, d.guard_triggered) == (path, guard), (name, op, n, k, build_n)
        assert d.c_cpu_est == c_cpu and d.c_gpu_est == c_gpu and d.gain == gain


def test_estimate_device_cost_matches_reference():
    for op, n, mode, est in G["estimate"]:
        pb = 188 if mode == FULL_ROW else None
        assert list(estimate_device_cost(op, n, 100, mode, pb)) == est


def test_calibrate_profile_matches_reference():
    c = G["calibrate_profile"]
    samples = [(n, TransferLedger(*vals)) for n, vals in c["samples"]]
    prof = calibrate_profile(samples)
    for k, v in c["profile"].items():
        assert getattr(prof, k) == pytest.approx(v, rel=1e-12)


def test_calibrate_cpu_model_matches_reference():
    c = G["calibrate_cpu"]
    model = calibrate_cpu_model([tuple(s) for s in c["samples"]])
    for k, v in c["model"].items():
        assert getattr(model, k) == pytest.approx(v, rel=1e-12)


def test_compute_stats_nearest_rank_matches_reference():
    for seq, med, p95, p99, mean in G["stats"]:
        s = compute_stats(seq)
        assert (s.median, s.p95, s.p99) == (med, p95, p99)
        assert s.mean == pytest.approx(mean, rel=1e-15)


def test_strict_gain_and_guard_rules():
    flat_cpu = CpuCostModel(0.0, 10e-3, 0.0, 10e-3)
    flat_dev = DeviceProfile(1e15, 1e15, 4e-3, 1e-15, 1e-15, 1e-15)
    cfg = GateConfig(cpu_model=flat_cpu, profile=flat_dev)
    assert decide(with_margin(cfg, 5e-3), OP_TOPK, 1000, 100).path == DEVICE
    assert decide(with_margin(cfg, 10e-3), OP_TOPK, 1000, 100).path == HOST
    d = decide(GateConfig(cpu_model=flat_cpu, profile=flat_dev, min_n_guard=5000), OP_TOPK, 1000, 100)
    assert d.guard_triggered and d.path == HOST
    # probes charge both sides to the device
    a = decide(GateConfig(), OP_PROBE, 1000, 1, None, 0).c_gpu_est
    b = decide(GateConfig(), OP_PROBE, 1000, 1, None, 10**6).c_gpu_est
    assert b > a


def test_validation_errors_like_the_reference():
    with pytest.raises(ValueError):
        GateConfig(margin_s=-1.0)
    with pytest.raises(ValueError):
        GateConfig(mode="bogus")
    with pytest.raises(ValueError):
        transfer_entry_bytes(FULL_ROW, None)
    with pytest.raises(ValueError):
        DeviceProfile(0.0, 1.0, 1.0, 1.0, 1.0, 1.0)
    with pytest.raises(ValueError):
        estimate_cpu_cost(DEFAULT_CPU_MODEL, "bogus", 10)
    with pytest.raises(CalibrationError):
        calibrate_profile([(10, TransferLedger.build(1, 1, 1.0, 1.0, 1.0, 1.0))] * 3)
    cfg = GateConfig.from_json_dict(GateConfig(margin_s=1e-3, min_n_guard=7).to_json_dict())
    assert cfg == GateConfig(margin_s=1e-3, min_n_guard=7)
    assert DeviceProfile.from_json_dict(DEFAULT_MODELED_PROFILE.to_json_dict()) == DEFAULT_MODELED_PROFILE


def test_modeled_e2e_speedup_at_3m_matches_reference_story():
    cmp = run_payload_comparison(WorkloadSpec(n_grid=(3_000_000,), repeats=1))
    full = next(r for r in cmp.e2e_rows if r.mode == FULL_ROW)
    key = next(r for r in cmp.e2e_rows if r.mode == KEY_ONLY)
    assert full.e2e_s == pytest.approx(2.4020016e-2, rel=1e-6)
    assert key.e2e_s == pytest.approx(1.942016e-3, rel=1e-6)
    assert key.speedup_vs_full_row == pytest.approx(12.368598, rel=1e-6)


def test_gated_mixed_workload_wins_the_tail_modeled():
    spec = WorkloadSpec(n_grid=(10_000, 1_000_000), repeats=250, mix=(0.8, 0.2), seed=3)
    host, device, gated = run_strategy_comparison(spec, GateConfig())
    hs, ds, gs = (compute_stats(r.all_samples()) for r in (host, device, gated))
    assert gs.p95 <= hs.p95 and gs.p95 <= ds.p95 and gs.p99 <= ds.p99
    assert 0.0 < gated.offload_rate < 1.0


class _LyingDevice(ModeledDevice):
    def topk(self, keys, k, mode=KEY_ONLY, payload_bytes=None):
        call = super().topk(keys, k, mode=mode, payload_bytes=payload_bytes)
        call.payload.rows[:] = call.payload.rows[::-1]
        return call


def test_divergent_answers_abort_the_comparison():
    spec = WorkloadSpec(n_grid=(1_000, 10_000), repeats=2)
    with pytest.raises(StrategyMismatchError):
        run_strategy_comparison(spec, GateConfig(), device=_LyingDevice())


def test_execute_gated_topk_and_probe_on_host_path():
    t = generate_table(5000, 16, seed=3)
    res, d, lat = execute_gated(t, OP_TOPK, 10, GateConfig())
    assert d.path == HOST and len(res) == 10 and lat > 0
    assert np.all(np.diff(res.keys) <= 0)
    res2, d2, _ = execute_gated((generate_table(300, 8, seed=1), t), OP_PROBE, 1, GateConfig())
    assert d2.path == HOST and res2.probe_count == 5000


def test_materialize_join_gathers_both_sides_in_pair_order():
    from paper_2601_19911_b200 import host_hash_build, host_hash_probe, extract_keys, materialize_join

    b = generate_table(2000, 12, seed=4)
    p = generate_table(5000, 7, seed=5)
    # small key domain so the tables actually join
    b = type(b)(np.floor(b.key_column / 2**45), b.payload_column)
    p = type(p)(np.floor(p.key_column / 2**45), p.payload_column)
    res = host_hash_probe(host_hash_build(extract_keys(b)), extract_keys(p))
    assert res.match_count > 100
    mj = materialize_join(b, p, res)
    assert len(mj) == res.match_count
    assert np.array_equal(mj.probe.keys, mj.build.keys)  # joined on equal keys
    assert np.array_equal(mj.build.payloads, b.payload_column[res.build_rows])
    assert np.array_equal(mj.probe.payloads, p.payload_column[res.probe_rows])
    bad = type(res)(np.array([0], np.uint32), np.array([10**6], np.uint32), 1)
    with pytest.raises(IndexError):
        materialize_join(b, p, bad)


def test_scaling_baseline_modeled_matches_reference():
    from paper_2601_19911_b200.harness import WorkloadSpec, run_scaling_baseline

    spec = WorkloadSpec(n_grid=(1_000, 100_000, 10**9), k=100, repeats=3)
    got = [list(r) for r in run_scaling_baseline(spec, backend="modeled")]
    assert got == gate_golden()["scaling_modeled"]


def test_scaling_baseline_host_wall_clock_rows():
    from paper_2601_19911_b200.harness import WorkloadSpec, run_scaling_baseline

    rows = run_scaling_baseline(WorkloadSpec(n_grid=(100, 2_000), k=10, repeats=2), backend="host")
    assert [(r.n, r.op) for r in rows] == [(100, "full_sort"), (100, "topk"), (2_000, "full_sort"), (2_000, "topk")]
    assert all(0 < r.median_s <= r.p95_s for r in rows)


# ---- opt-in K-aware host cost terms (not in the reference; defaults keep its model) ----


def test_k_aware_fields_default_to_the_reference_model():
    m = CpuCostModel(1e-10, 5e-6, 5e-10, 5e-6)
    assert not m.k_aware
    assert set(m.to_json_dict()) == {"alpha_sort", "beta_sort", "alpha_match", "beta_match"}
    for op, n, k in ((OP_TOPK, 10**6, 10**5), (OP_PROBE, 10**4, 500)):
        ref = (1e-10 * n * math.log2(n) + 5e-6) if op == OP_TOPK else (5e-10 * n * k + 5e-6)
        assert estimate_cpu_cost(m, op, n, k) == ref
    ext = CpuCostModel(1e-10, 5e-6, 5e-10, 5e-6, alpha_topk_k=3e-9, alpha_pair=2e-9)
    assert ext.k_aware and CpuCostModel.from_json_dict(ext.to_json_dict()) == ext
    assert CpuCostModel.from_json_dict(m.to_json_dict()) == m
    with pytest.raises(ValueError):
        CpuCostModel(1e-10, 5e-6, 5e-10, 5e-6, alpha_pair=-1.0)


def test_k_aware_estimates():
    ext = CpuCostModel(1e-10, 5e-6, 5e-10, 5e-6, alpha_topk_k=3e-9, alpha_pair=2e-9)
    n, k = 10**6, 10**5
    assert estimate_cpu_cost(ext, OP_TOPK, n, k) == pytest.approx(
        1e-10 * n * math.log2(n) + 3e-9 * k * math.log2(k) + 5e-6, rel=1e-15)
    # K is clamped to n: K >= n costs what K = n costs
    assert estimate_cpu_cost(ext, OP_TOPK, 1000, 10**6) == estimate_cpu_cost(ext, OP_TOPK, 1000, 1000)
    # probes are linear in n and M instead of n * M
    assert estimate_cpu_cost(ext, OP_PROBE, 1000, 500) == pytest.approx(5e-10 * 1000 + 2e-9 * 500 + 5e-6)


def test_k_aware_calibration_recovers_the_generating_constants():
    a_s, a_k, b_s, a_m, a_p, b_m = 4e-11, 2e-9, 3e-6, 7e-9, 1.5e-8, 4e-6
    samples = []
    for n in (10**4, 10**5, 10**6, 4 * 10**6):
        for k in (10, 1000, 10**5):
            kk = min(k, n)
            samples.append((OP_TOPK, n, k, a_s * n * math.log2(n) + a_k * kk * math.log2(max(kk, 2)) + b_s))
    for n in (10**4, 10**5, 10**6):
        for m in (1, n // 2):
            samples.append((OP_PROBE, n, m, a_m * n + a_p * m + b_m))
    got = calibrate_cpu_model(samples, k_aware=True)
    for name, want in (("alpha_sort", a_s), ("alpha_topk_k", a_k), ("beta_sort", b_s), ("alpha_match", a_m),
                       ("alpha_pair", a_p), ("beta_match", b_m)):
        assert getattr(got, name) == pytest.approx(want, rel=1e-6), name
    # the reference fit of the same samples is unchanged by the option
    assert not calibrate_cpu_model(samples).k_aware


def test_k_aware_calibration_needs_two_k_values():
    samples = [(OP_TOPK, n, 100, 1e-9 * n) for n in (10**4, 10**5, 10**6)]
    with pytest.raises(CalibrationError):
        calibrate_cpu_model(samples, k_aware=True)
    assert calibrate_cpu_model(samples).alpha_sort > 0.0


def test_k_aware_gate_fixes_the_reference_forms_misses():
    """The two miss patterns of profiles/r1_gate_cells.json: Top-K with a large K
    stays on the host under n*log(n), and a tiny probe with a large M goes to the
    device under n*M. The K-aware terms move both the other way."""
    prof = DeviceProfile(5e10, 5e10, 5e-5, 1e-12, 1e-12, 1e-9)
    ref = CpuCostModel(4.3e-11, 0.0, 7.8e-9, 0.0)
    ext = CpuCostModel(4.3e-11, 0.0, 7.8e-9, 0.0, alpha_topk_k=6e-9, alpha_pair=1e-9)
    n, k = 10**5, 10**5
    assert decide(GateConfig(cpu_model=ref, profile=prof), OP_TOPK, n, k).path == HOST
    assert decide(GateConfig(cpu_model=ext, profile=prof), OP_TOPK, n, k).path == DEVICE
    assert decide(GateConfig(cpu_model=ref, profile=prof), OP_PROBE, 1000, 500, None, 100).path == DEVICE
    assert decide(GateConfig(cpu_model=ext, profile=prof), OP_PROBE, 1000, 500, None, 100).path == HOST


def test_materialize_joins_on_the_query_path_cpu():
    """GateConfig(materialize_joins=True): the probe query returns both sides
    gathered in pair order, on the modeled (virtual-clock) device and the host path."""
    from paper_2601_19911_b200 import DEVICE, HOST, OP_PROBE, GateConfig, ModeledDevice, execute_path, generate_table
    from paper_2601_19911_b200.store import ColumnTable, MaterializedJoin

    bt, pt = generate_table(300, 4, seed=3), generate_table(2_000, 4, seed=4)
    # the probe table starts with the build keys, so that pairs exist
    pt = ColumnTable(np.concatenate([bt.key_column, pt.key_column])[:2_000], pt.payload_column, 4)
    for path in (DEVICE, HOST):
        res, lat = execute_path((bt, pt), OP_PROBE, 1, GateConfig(materialize_joins=True), ModeledDevice(), path)
        assert isinstance(res, MaterializedJoin) and len(res) >= 300 and lat > 0
        assert np.array_equal(res.probe.keys, res.build.keys)
        assert np.array_equal(res.probe.payloads, pt.payload_column[res.probe.row_ids])
        assert np.array_equal(res.build.payloads, bt.payload_column[res.build.row_ids])


def test_cli_bench_modeled_writes_golp_style_outputs(tmp_path):
    """`cli bench` (golp bench's shape, pkg/src/golp/cli.py:183-237) on the modeled backend."""
    import json

    from paper_2601_19911_b200 import cli

    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"workload": {"n_grid": [1_000, 10_000, 100_000], "repeats": 2, "payload_bytes": 16},
                               "gpus": 1}))
    assert cli.main(["bench", "--config", str(cfg), "--backend", "modeled", "--out", str(tmp_path / "out")]) == 0
    summary = json.loads((tmp_path / "out" / "summary.json").read_text())
    assert summary["backend"] == "modeled" and set(summary["strategies"]) == {"host_only", "device_always", "gated"}
    for f in ("scaling.csv", "payload.csv", "transfer.csv", "e2e.csv", "strategies.csv"):
        assert (tmp_path / "out" / f).read_text().count("\n") > 1
    assert cli.main(["bench", "--backend", "modeled", "--gpus", "0", "--out", str(tmp_path / "o2")]) == 2


def test_table_dump_round_trip_and_reference_format(tmp_path):
    """save_table / load_table in the reference's dump format (store.py:214-244):
    byte-identical files, and each side loads the other's dumps."""
    import sys
    from pathlib import Path

    from paper_2601_19911_b200 import store

    t = store.generate_table(5_000, 12, seed=9)
    ours = tmp_path / "ours.golp"
    store.save_table(t, ours)
    for mapped in (True, False):
        back = store.load_table(ours, mapped=mapped)
        assert back.seed == t.seed and np.array_equal(back.key_column, t.key_column)
        assert np.array_equal(back.payload_column, t.payload_column)
        assert not back.key_column.flags.writeable
    bad = tmp_path / "bad.golp"
    bad.write_bytes(ours.read_bytes()[:-1])
    with pytest.raises(ValueError):
        store.load_table(bad)
    ref = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
    if not (ref / "golp").exists():
        pytest.skip("reference golp not installed (baseline/install_reference.sh)")
    sys.path.insert(0, str(ref))
    import golp.store as gs

    theirs = tmp_path / "theirs.golp"
    gs.save_table(gs.generate_table(5_000, 12, seed=9), theirs)
    assert theirs.read_bytes() == ours.read_bytes()
    g = gs.load_table(ours)
    assert np.array_equal(g.key_column, t.key_column) and np.array_equal(g.payload_column, t.payload_column)
