"""Reference acceptance criterion 7 (pkg/tests/test_acceptance.py:252-270) on the
B200: the 500-query 80/20 stream (n in {1e4, 1e6}, seed 3, 188-B payloads) under
host_only / device_always / gated, P50/P95/P99 per strategy and per n.

python tools/crit7.py [RUNS] [--calibrated]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import B200Device, GateConfig  # noqa: E402
from paper_2601_19911_b200.harness import WorkloadSpec, calibrate_device_profile, compute_stats, run_strategy_comparison  # noqa: E402

import gc
if "--nogc" in sys.argv:
    gc.disable()
runs = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 3
spec = WorkloadSpec(n_grid=(10_000, 1_000_000), repeats=250, mix=(0.8, 0.2), seed=3)
out = []
with B200Device() as dev:
    cfg = GateConfig()
    if "--calibrated" in sys.argv:
        cfg = GateConfig(profile=calibrate_device_profile(dev))
    tables = {}
    for r in range(runs):
        host, device, gated = run_strategy_comparison(spec, cfg, device=dev, tables=tables)
        row = {}
        for run in (host, device, gated):
            st = compute_stats(run.all_samples())
            row[run.strategy] = {"p50_ms": st.median * 1e3, "p95_ms": st.p95 * 1e3, "p99_ms": st.p99 * 1e3,
                                 "per_n": {n: {"p50_ms": s.median * 1e3, "p95_ms": s.p95 * 1e3} for n, s in
                                           run.per_n.items()}, "offload_rate": run.offload_rate}
        ok = (row["gated"]["p95_ms"] <= row["host_only"]["p95_ms"] and row["gated"]["p95_ms"] <= row["device_always"]["p95_ms"]
              and row["gated"]["p99_ms"] <= row["device_always"]["p99_ms"])
        row["pass"] = ok
        out.append(row)
        print(json.dumps({s: {k: round(v, 4) for k, v in row[s].items() if k.endswith("_ms")} for s in
                          ("host_only", "device_always", "gated")}), "PASS" if ok else "FAIL", flush=True)
print(json.dumps(out))
