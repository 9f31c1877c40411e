"""Config C5 (BASELINE.json) cell by cell on the B200: for every (op, N, K or M,
mode) cell, P50/P95/P99 of end-to-end query latency (extract_keys + path +
materialize, gate.execute_path semantics, pkg/src/golp/gate.py:167-233) for
CPU-only (the host engine), always-on offload (B200Device) and the Risky Gate
(execute_gated with the calibrated profile / CPU model), plus the gate's choice.

    python tools/gate_cells.py [out.json] [--max-n N]      (N up to 1e9; full-row cells to 1e7)

The DeviceProfile is calibrated from B200 ledgers and the CpuCostModel from
host-engine timings in the same run (tools/gate_sweep.py does the same); the
gate then decides each cell with those constants. Repeats shrink with N so the
whole sweep stays within a few minutes; percentiles are nearest-rank
(pkg/src/golp/harness.py:127-143)."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2601_19911_b200 import (  # noqa: E402
    B200Device, FULL_ROW, KEY_ONLY, OP_PROBE, OP_TOPK, GateConfig, calibrate_cpu_model, host_topk,
    random_key_vector)
from paper_2601_19911_b200.gate import DEVICE, HOST, execute_gated, execute_path  # noqa: E402
from paper_2601_19911_b200.harness import calibrate_device_profile, compute_stats, table_seed  # noqa: E402
from paper_2601_19911_b200.errors import CapacityError  # noqa: E402
from paper_2601_19911_b200.host import host_hash_build, host_hash_probe  # noqa: E402
from paper_2601_19911_b200.store import ColumnTable, extract_keys, generate_table  # noqa: E402


# A query stream does not call the host engine back to back: its worker pool has gone
# idle (spin, then futex sleep) by the next query. The K-aware calibration idles this
# long before each timed host query so it pays the same wake-up as the cells do.
IDLE_S = 0.002


def repeats_for(n):
    return 25 if n <= 100_000 else (11 if n <= 1_000_000 else (5 if n <= 10_000_000 else (3 if n <= 100_000_000 else 2)))


def stats(ts):
    s = compute_stats(ts)
    return {"p50": s.median, "p95": s.p95, "p99": s.p99}


def probe_tables(n, payload, seed):
    """Probe side of n rows, build side n/10 rows, keys uniform in [0, 2 * build):
    ~0.5 matches per probe (BASELINE's join shape)."""
    nb = max(1, n // 10)
    rng = np.random.Generator(np.random.PCG64(seed))
    bk = rng.integers(0, 2 * nb, nb).astype(np.float64)
    pk = rng.integers(0, 2 * nb, n).astype(np.float64)
    pay = lambda m: np.zeros((m, payload), dtype=np.uint8)  # noqa: E731
    return ColumnTable(bk, pay(nb), seed), ColumnTable(pk, pay(n), seed + 1)


def run_cell(tables, op, k, cfg, dev, reps, cfg_k=None):
    """Warm each path twice (B200Device page-locks a reused input column on its
    second call, a one-off ~0.1-0.4 s at 1e8 rows that a query stream amortizes),
    then interleave host / device / gated per repeat. A host path the reference
    itself refuses (host_hash_build's 2 GiB table budget, host.py:155-159, from
    ~9.4e7 build rows) is reported as such and not timed."""
    host_ok = True
    try:
        execute_path(tables, op, k, cfg, dev, HOST)
    except CapacityError as e:
        host_ok = False
        host_err = f"CapacityError: {e}"
    for _ in range(2):
        for path in ((HOST, DEVICE) if host_ok else (DEVICE,)):
            execute_path(tables, op, k, cfg, dev, path)
    host, devt, gated, gated_k = [], [], [], []
    choice = choice_k = None
    for _ in range(reps):
        if host_ok:
            host.append(execute_path(tables, op, k, cfg, dev, HOST)[1])
        devt.append(execute_path(tables, op, k, cfg, dev, DEVICE)[1])
        _, decision, t = execute_gated(tables, op, k, cfg, dev)
        gated.append(t)
        choice = decision.path
        if cfg_k is not None:
            _, decision, t = execute_gated(tables, op, k, cfg_k, dev)
            gated_k.append(t)
            choice_k = decision.path
    out = {"cpu_only": stats(host) if host_ok else {"error": host_err}, "always_on": stats(devt),
           "gated": stats(gated), "gate_choice": choice, "repeats": reps}
    if cfg_k is not None:
        out.update({"gated_k_aware": stats(gated_k), "gate_choice_k_aware": choice_k})
    return out


def main(out_path, max_n):
    t0 = time.time()
    dev = B200Device()
    prof = calibrate_device_profile(dev, ns=(100_000, 1_000_000, 4_000_000, 16_000_000), repeats=3,
                                    probe_ns=(200_000, 2_000_000, 8_000_000))
    samples = []
    for n in (100_000, 1_000_000, 4_000_000, 16_000_000):  # host Top-K (sort family)
        kv = random_key_vector(n, n)
        host_topk(kv, 100)
        samples.append((OP_TOPK, n, 100, _time(lambda: host_topk(kv, 100))))
    # host probe (match family). The reference's form is alpha_match * n * k + beta
    # (pkg/src/golp/gate.py:37-160); a hash join's host cost grows with n alone, so
    # the samples pass k = 1 and alpha_match comes out per probe. Cells with M = 1
    # are then the well-posed gate; cells with M = expected matches show what the
    # n * M form does with that constant.
    for n in (100_000, 1_000_000, 4_000_000):
        b, p = probe_tables(n, 1, n)
        bkv, pkv = extract_keys(b), extract_keys(p)
        samples.append((OP_PROBE, n, 1, _time(lambda: host_hash_probe(host_hash_build(bkv), pkv))))
    cpu = calibrate_cpu_model(samples)
    # K-aware extension (CpuCostModel.alpha_topk_k / alpha_pair; not the reference's
    # form), calibrated on the query the gate decides: execute_path's host wall time
    # (extract_keys + engine + materialize), not the bare engine call. Top-K samples at
    # several K; probe samples at two match rates so that n and M separate (the second
    # probe side draws its keys outside the build domain, M = 0).
    k_samples = []
    cfg_h = GateConfig(profile=prof, cpu_model=cpu)
    for n in (1_000, 10_000, 100_000, 1_000_000, 4_000_000, 16_000_000):
        t = generate_table(n, payload_bytes=1, seed=table_seed(5, n), memory_budget=1 << 40)
        for k in (10, 1000, 100_000):
            k_samples.append((OP_TOPK, n, k, _time(lambda: execute_path(t, OP_TOPK, k, cfg_h, dev, HOST),
                                                   9 if n <= 10_000 else 3, IDLE_S)))
    for n in (1_000, 10_000, 100_000, 1_000_000, 4_000_000):
        b, p = probe_tables(n, 1, n)
        m = len(host_hash_probe(host_hash_build(extract_keys(b)), extract_keys(p)).probe_rows)
        k_samples.append((OP_PROBE, n, m, _time(lambda: execute_path((b, p), OP_PROBE, 1, cfg_h, dev, HOST),
                                                9 if n <= 10_000 else 3, IDLE_S)))
        miss = ColumnTable(p.key_column + 4.0 * b.row_count, p.payload_column, n + 1)
        k_samples.append((OP_PROBE, n, 0, _time(lambda: execute_path((b, miss), OP_PROBE, 1, cfg_h, dev, HOST),
                                                9 if n <= 10_000 else 3, IDLE_S)))
    cpu_k = calibrate_cpu_model(k_samples, k_aware=True)
    # The profile is fitted on call ledgers, which leave out the per-query host work
    # around the call (extract_keys, materialize, Python). The K-aware gate charges it
    # as its margin: the smallest device query's wall time minus its modeled cost.
    small = generate_table(1_000, payload_bytes=1, seed=3, memory_budget=1 << 40)
    cfg0 = GateConfig(profile=prof, cpu_model=cpu_k)
    for _ in range(3):
        execute_path(small, OP_TOPK, 10, cfg0, dev, DEVICE)
    wall = sorted(execute_path(small, OP_TOPK, 10, cfg0, dev, DEVICE)[1] for _ in range(9))[4]
    margin_k = max(0.0, wall - execute_gated(small, OP_TOPK, 10, cfg0, dev)[1].c_gpu_est)
    cells = []
    ns = [n for n in (1_000, 10_000, 100_000, 1_000_000, 10_000_000, 100_000_000, 1_000_000_000) if n <= max_n]
    for n in ns:
        for mode in (KEY_ONLY, FULL_ROW):
            if mode == FULL_ROW and n > 10_000_000:
                continue  # 196 B/row: 19.6 GB per call at 1e8 -- host RAM, not the device, is the limit
            payload = 188 if mode == FULL_ROW else 1  # key-only never ships the payload
            cfg = GateConfig(mode=mode, profile=prof, cpu_model=cpu)
            cfg_k = GateConfig(mode=mode, profile=prof, cpu_model=cpu_k, margin_s=margin_k)
            table = generate_table(n, payload_bytes=payload, seed=table_seed(7, n),
                                   memory_budget=1 << 40)
            for k in (10, 1000, 100_000):
                if k > n:
                    continue
                cell = {"op": OP_TOPK, "n": n, "k": k, "mode": mode}
                cell.update(run_cell(table, OP_TOPK, k, cfg, dev, repeats_for(n), cfg_k))
                cells.append(cell)
                print(json.dumps(cell), flush=True)
            del table
            tables = probe_tables(n, payload, table_seed(9, n))
            for m in (1, n // 2):  # the gate's M: a point estimate and the expected match count
                cell = {"op": OP_PROBE, "n": n, "build_n": tables[0].row_count, "m": m, "mode": mode}
                cell.update(run_cell(tables, OP_PROBE, max(m, 1), cfg, dev, repeats_for(n), cfg_k))
                cells.append(cell)
                print(json.dumps(cell), flush=True)
    # per cell, how the gate's percentiles compare with the better fixed strategy
    for c in cells:
        for q in ("p95", "p99"):
            best = min(c["cpu_only"].get(q, float("inf")), c["always_on"][q])
            c[f"gated_{q}_over_best_fixed"] = c["gated"][q] / best if best > 0 else None
            c[f"gated_k_aware_{q}_over_best_fixed"] = c["gated_k_aware"][q] / best if best > 0 else None
    out = {"profile_b200": prof.to_json_dict(), "cpu_model_host_engine": cpu.to_json_dict(),
           "cpu_model_host_engine_k_aware": cpu_k.to_json_dict(), "margin_s_k_aware": margin_k, "cells": cells, "wall_s": time.time() - t0}
    Path(out_path).write_text(json.dumps(out, indent=1))
    dev.close()


def _time(fn, reps=3, idle_s=0.0):
    ts = []
    for _ in range(reps):
        if idle_s:
            time.sleep(idle_s)
        a = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - a)
    return sorted(ts)[len(ts) // 2]


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    max_n = 1_000_000_000
    if "--max-n" in sys.argv:
        max_n = int(float(sys.argv[sys.argv.index("--max-n") + 1]))
    main(args[0] if args else "gpurun_out/gate_cells.json", max_n)
