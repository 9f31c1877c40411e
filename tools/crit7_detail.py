"""Large-query (n=1e6) latencies of crit 7's stream under device_always vs gated,
split by what ran just before (host or device query)."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import DEVICE, HOST, OP_TOPK, B200Device, GateConfig, execute_gated, execute_path, generate_table  # noqa: E402
from paper_2601_19911_b200.harness import WorkloadSpec, query_sizes, table_seed  # noqa: E402

spec = WorkloadSpec(n_grid=(10_000, 1_000_000), repeats=250, mix=(0.8, 0.2), seed=3)
tables = {n: generate_table(n, spec.payload_bytes, seed=table_seed(spec.seed, n)) for n in spec.n_grid}
sizes = query_sizes(spec)
cfg = GateConfig()
with B200Device() as dev:
    for n in spec.n_grid:
        for _ in range(3):
            execute_path(tables[n], OP_TOPK, 100, cfg, dev, DEVICE)
            execute_path(tables[n], OP_TOPK, 100, cfg, dev, HOST)
    for rep in range(2):
        for strat in ("device_always", "gated"):
            lat = {HOST: [], DEVICE: []}
            prev = DEVICE
            for n in sizes:
                if strat == "gated":
                    _, d, t = execute_gated(tables[n], OP_TOPK, 100, cfg, dev)
                    path = d.path
                else:
                    _, t = execute_path(tables[n], OP_TOPK, 100, cfg, dev, DEVICE)
                    path = DEVICE
                if n == 1_000_000:
                    lat[prev].append(t * 1e3)
                prev = path
            for p, xs in lat.items():
                if xs:
                    xs.sort()
                    print(f"{strat:14s} after {p:6s}: n={len(xs):3d} p50 {statistics.median(xs):.4f} p75 {xs[int(.75*len(xs))]:.4f} p95 {xs[int(.95*len(xs))]:.4f} ms")
