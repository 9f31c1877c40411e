"""Config C5 (BASELINE.json): Risky Gate sweep on the B200. Calibrates the
DeviceProfile from B200 ledgers and the CpuCostModel from host-engine timings,
then reports decide() under the reference's default constants next to the
calibrated ones over N x K x mode, and P50/P95/P99 of host_only /
device_always / gated on the reference's 80/20 mixed stream (crit 7 shape).

    python tools/gate_sweep.py [out.json]
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2601_19911_b200 import (  # noqa: E402
    B200Device, FULL_ROW, KEY_ONLY, OP_PROBE, OP_TOPK, GateConfig, KeyVector, calibrate_cpu_model, decide,
    host_hash_build, host_hash_probe, host_topk, random_key_vector)
from paper_2601_19911_b200.harness import (  # noqa: E402
    WorkloadSpec, calibrate_device_profile, compute_stats, run_strategy_comparison)


def main(out_path):
    dev = B200Device()
    t0 = time.time()
    prof = calibrate_device_profile(dev, ns=(100_000, 1_000_000, 4_000_000, 16_000_000), repeats=3,
                                    probe_ns=(200_000, 2_000_000, 8_000_000))
    cpu_samples = []
    for n in (100_000, 1_000_000, 4_000_000, 16_000_000):
        kv = random_key_vector(n, n)
        host_topk(kv, 100)
        ts = []
        for _ in range(3):
            a = time.perf_counter()
            host_topk(kv, 100)
            ts.append(time.perf_counter() - a)
        cpu_samples.append((OP_TOPK, n, 100, sorted(ts)[1]))
    # host-engine probes: probe side n, build n/10, keys in [0, n/5) (~0.5 matches per probe)
    for n in (100_000, 1_000_000, 4_000_000):
        rng = np.random.default_rng(n)
        nb = n // 10
        b = KeyVector(rng.integers(0, n // 5, nb).astype(np.float64), np.arange(nb, dtype=np.uint32))
        p = KeyVector(rng.integers(0, n // 5, n).astype(np.float64), np.arange(n, dtype=np.uint32))
        host_hash_probe(host_hash_build(b), p)
        ts = []
        for _ in range(3):
            a = time.perf_counter()
            host_hash_probe(host_hash_build(b), p)
            ts.append(time.perf_counter() - a)
        cpu_samples.append((OP_PROBE, n, 1, sorted(ts)[1]))
    cpu = calibrate_cpu_model(cpu_samples)
    ref_cfg = GateConfig()
    cal_cfg = GateConfig(profile=prof, cpu_model=cpu)
    grid = []
    for n in (1_000, 10_000, 20_000, 100_000, 1_000_000, 10_000_000, 100_000_000, 1_000_000_000):
        for k in (10, 100, 1000, 100_000):
            for mode in (KEY_ONLY, FULL_ROW):
                pb = 188 if mode == FULL_ROW else None
                r = decide(GateConfig(mode=mode), OP_TOPK, n, k, pb)
                c = decide(GateConfig(mode=mode, profile=prof, cpu_model=cpu), OP_TOPK, n, k, pb)
                grid.append({"n": n, "k": k, "mode": mode, "reference_decision": r.path, "reference_gain_s": r.gain,
                             "calibrated_decision": c.path, "calibrated_gain_s": c.gain,
                             "c_gpu_calibrated_s": c.c_gpu_est, "c_cpu_calibrated_s": c.c_cpu_est})
    # the M axis: probes of n keys against a build side of n/10, M (passed as k,
    # the reference's per-probe factor in C_cpu and match count in C_gpu,
    # gate.py:127-128 / device.py:172-175) = 1 or the expected n/2 matches
    probe_grid = []
    for n in (1_000, 10_000, 20_000, 100_000, 1_000_000, 10_000_000, 100_000_000, 1_000_000_000):
        for m in (1, max(1, n // 2)):
            for mode in (KEY_ONLY, FULL_ROW):
                pb = 188 if mode == FULL_ROW else None
                r = decide(GateConfig(mode=mode), OP_PROBE, n, m, pb, build_n=n // 10)
                c = decide(GateConfig(mode=mode, profile=prof, cpu_model=cpu), OP_PROBE, n, m, pb, build_n=n // 10)
                probe_grid.append({"n_probe": n, "n_build": n // 10, "m": m, "mode": mode,
                                   "reference_decision": r.path, "reference_gain_s": r.gain,
                                   "calibrated_decision": c.path, "calibrated_gain_s": c.gain,
                                   "c_gpu_calibrated_s": c.c_gpu_est, "c_cpu_calibrated_s": c.c_cpu_est})
    strat = {}
    # crit 7's exact stream (pkg/tests/test_acceptance.py:252-270): 500 queries,
    # 80/20 over n in {1e4, 1e6}, seed 3, 188-byte payloads; three runs each
    spec = WorkloadSpec(n_grid=(10_000, 1_000_000), repeats=250, mix=(0.8, 0.2), seed=3)
    tables = {}
    for label, cfg in (("reference_constants", ref_cfg), ("calibrated", cal_cfg)):
        strat[label] = []
        for _ in range(3):
            runs = run_strategy_comparison(spec, cfg, device=dev, tables=tables)
            strat[label].append({r.strategy: {**{k: getattr(compute_stats(r.all_samples()), k)
                                                 for k in ("median", "p95", "p99")},
                                              "offload_rate": r.offload_rate} for r in runs})
    # the paper's key-only vs full-row experiment on the B200:
    # Top-K K=100, payload 188 B; E2E full-row = h2d+kernel+d2h, key-only = whole
    # ledger incl. late materialization (run_payload_comparison semantics)
    from paper_2601_19911_b200.harness import run_payload_comparison

    pay = run_payload_comparison(WorkloadSpec(n_grid=(1_000_000, 3_000_000, 10_000_000), repeats=1, k=100,
                                              payload_bytes=188), device=dev)
    pay = run_payload_comparison(WorkloadSpec(n_grid=(1_000_000, 3_000_000, 10_000_000), repeats=1, k=100,
                                              payload_bytes=188), device=dev)  # second pass: warm
    payload = {"transfer": [r._asdict() for r in pay.transfer_rows], "e2e": [r._asdict() for r in pay.e2e_rows],
               "transfer_time_ratio_full_over_key": {
                   str(n): next(r.transfer_s for r in pay.payload_rows if r.n == n and r.mode == FULL_ROW) /
                   next(r.transfer_s for r in pay.payload_rows if r.n == n and r.mode == KEY_ONLY)
                   for n in (1_000_000, 3_000_000, 10_000_000)}}
    out = {"profile_b200": prof.to_json_dict(), "cpu_model_host_engine": cpu.to_json_dict(),
           "decisions": grid, "probe_decisions": probe_grid, "strategy_80_20_stream": strat, "key_only_vs_full_row": payload,
           "wall_s": time.time() - t0}
    Path(out_path).write_text(json.dumps(out, indent=1))
    print(json.dumps({"profile": out["profile_b200"], "strategies": strat,
                      "payload_ratio": payload["transfer_time_ratio_full_over_key"],
                      "e2e_speedup": [(r["n"], r["mode"], r["speedup_vs_full_row"]) for r in payload["e2e"]]},
                     indent=1))
    dev.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gate_sweep.json")
