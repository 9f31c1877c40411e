"""`python -m paper_2601_19911_b200.cli bench`: the reference's `golp bench` run
(pkg/src/golp/cli.py:183-237) on the offload path this package rebuilds, with
the B200 backend registered next to the modeled one.

    python -m paper_2601_19911_b200.cli bench [--config cfg.json] [--backend b200|modeled]
                                             [--gpus G] [--out DIR] [--seed S]

The config is golp's JSON form ({"workload": {n_grid, k, repeats, payload_bytes,
mix, seed}, "gate": {...}, "backend": ..., "gpus": G, "memory_budget": bytes|null,
"output_dir": ...}); `gpus` shards every device call over G GPUs of this
process and `memory_budget: null` lifts the 2 GiB table cap for large-N
key-only runs (store.py:152-157). With the b200 backend the gate is calibrated
on this box (host-engine CpuCostModel from the scaling rows, DeviceProfile from
CUDA-event-timed B200 calls, one profile per G) before the strategy comparison.

Written files (CSV + summary.json, the subset of golp's export_report,
harness.py:545-620, that the offload path produces): scaling.csv (fig3 rows:
host full_sort / topk and, for b200, the same ops through the device),
payload.csv / transfer.csv / e2e.csv (key-only vs full-row, fig4/6/7),
strategies.csv (P50/P95/P99 of host_only / device_always / gated, fig5),
summary.json. Break-even fitting and margin sweeps stay with golp
(DESIGN.md §10). Exit codes as golp: 0 ok, 2 usage / input errors.
"""

from __future__ import annotations

import argparse
import csv
import dataclasses
import json
import sys
from pathlib import Path

from .device import KEY_ONLY, make_device
from .errors import GolpError
from .gate import OP_FULL_SORT, GateConfig, calibrate_cpu_model
from .harness import (WorkloadSpec, calibrate_device_profile, compute_stats, run_payload_comparison,
                      run_scaling_baseline, run_strategy_comparison)

EXIT_OK = 0
EXIT_USAGE = 2
BACKENDS = ("modeled", "b200")
_WORKLOAD_KEYS = ("n_grid", "k", "repeats", "payload_bytes", "mix", "seed")


def _write_csv(path: Path, header: list, rows) -> Path:
    with open(path, "w", newline="", encoding="utf-8") as f:
        w = csv.writer(f)
        w.writerow(header)
        w.writerows(rows)
    return path


def load_config(args) -> dict:
    raw = json.loads(Path(args.config).read_text(encoding="utf-8")) if args.config else {}
    if not isinstance(raw, dict):
        raise ValueError("config must hold a JSON object")
    wl = {k: v for k, v in dict(raw.get("workload") or {}).items() if k in _WORKLOAD_KEYS}
    if "n_grid" in wl:
        wl["n_grid"] = tuple(wl["n_grid"])
    if wl.get("mix") is not None:
        wl["mix"] = tuple(wl["mix"])
    if args.seed is not None:
        wl["seed"] = args.seed
    if "memory_budget" in raw:
        wl["memory_budget"] = raw["memory_budget"]
    backend = args.backend or raw.get("backend") or "b200"
    if backend not in BACKENDS:
        raise ValueError(f"backend must be one of {BACKENDS}, got {backend!r}")
    gpus = int(args.gpus if args.gpus is not None else raw.get("gpus", 1))
    if gpus < 1:
        raise ValueError("gpus must be >= 1")
    return {"spec": WorkloadSpec(**wl), "gate": GateConfig.from_json_dict(raw.get("gate") or {}),
            "backend": backend, "gpus": gpus, "out": Path(args.out or raw.get("output_dir") or "golp_out")}


def cmd_bench(args) -> int:
    cfg = load_config(args)
    spec, gate, out = cfg["spec"], cfg["gate"], cfg["out"]
    out.mkdir(parents=True, exist_ok=True)
    device = make_device(cfg["backend"], gate.profile, gpus=cfg["gpus"])
    try:
        if cfg["backend"] == "b200":
            scaling = run_scaling_baseline(spec, backend="host", device=device)
            cpu = calibrate_cpu_model([(OP_FULL_SORT, r.n, spec.k, r.median_s) for r in scaling
                                       if r.op == OP_FULL_SORT])
            profile = calibrate_device_profile(device)
            gate = dataclasses.replace(gate, cpu_model=cpu, profile=profile)
        else:
            scaling = run_scaling_baseline(spec, backend="modeled", cpu_model=gate.cpu_model)
        payload = run_payload_comparison(spec, device=device)
        strategies = run_strategy_comparison(spec, gate, device=device)
    finally:
        device.close()
    files = [
        _write_csv(out / "scaling.csv", ["n", "op", "median_s", "p95_s"], [tuple(r) for r in scaling]),
        _write_csv(out / "payload.csv", ["n", "mode", "bytes", "transfer_s"], [tuple(r) for r in payload.payload_rows]),
        _write_csv(out / "transfer.csv", ["n", "mode", "h2d_bytes", "t_h2d", "t_kernel", "t_d2h", "t_post", "total_s"],
                   [tuple(r) for r in payload.transfer_rows]),
        _write_csv(out / "e2e.csv", ["n", "mode", "e2e_s", "speedup_vs_full_row"], [tuple(r) for r in payload.e2e_rows]),
        _write_csv(out / "strategies.csv", ["strategy", "n", "median_s", "p95_s", "p99_s", "offload_rate"],
                   [(run.strategy, n, st.median, st.p95, st.p99, run.offload_rate)
                    for run in strategies for n, st in sorted(run.per_n.items())]),
    ]
    overall = {run.strategy: dataclasses.asdict(compute_stats(run.all_samples())) for run in strategies}
    for v in overall.values():
        v.pop("samples", None)
    summary = {"backend": cfg["backend"], "gpus": cfg["gpus"], "workload": dataclasses.asdict(spec),
               "gate": gate.to_json_dict(), "strategies": overall,
               "key_only_speedup": {str(r.n): r.speedup_vs_full_row for r in payload.e2e_rows if r.mode == KEY_ONLY},
               "files": [p.name for p in files]}
    files.append(out / "summary.json")
    files[-1].write_text(json.dumps(summary, indent=1, default=str), encoding="utf-8")
    for p in files:
        print(f"wrote {p}")
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2601_19911_b200.cli")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="scaling / payload / strategy runs, CSV + summary.json")
    b.add_argument("--config")
    b.add_argument("--backend", choices=BACKENDS)
    b.add_argument("--gpus", type=int)
    b.add_argument("--out")
    b.add_argument("--seed", type=int)
    args = ap.parse_args(argv)
    try:
        return cmd_bench(args)
    except (GolpError, ValueError, OSError) as e:  # golp's cli.py:423-425 mapping
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
