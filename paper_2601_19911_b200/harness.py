"""Strategy comparison and latency statistics for the Risky Gate (the P95/P99
producer), plus the key-only vs full-row payload comparison.

Restates the parts of the reference harness that sit on the offload path
(pkg/src/golp/harness.py:127-143 compute_stats, :228-239 query_sizes / table
seeds, :290-325 run_payload_comparison, :335-435 run_strategy_comparison) and
adds `calibrate_device_profile`, which turns measured B200 ledgers into the
gate's DeviceProfile. Figure export, margin sweeps and break-even fitting stay
with golp (out of scope).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass
from typing import NamedTuple, Optional, Sequence

import numpy as np

from .device import (DEFAULT_MODELED_PROFILE, FULL_ROW, KEY_ONLY, OP_PROBE, OP_TOPK, ModeledDevice, TransferLedger,
                     calibrate_profile)
from .errors import StrategyMismatchError
from .gate import DEFAULT_CPU_MODEL, DEVICE, HOST, OP_FULL_SORT, GateConfig, estimate_cpu_cost, execute_gated, execute_path
from .host import host_full_sort, host_topk, mix64
from .store import DEFAULT_MEMORY_BUDGET, DEFAULT_PAYLOAD_BYTES, ColumnTable, generate_table, random_key_vector

HOST_ONLY = "host_only"
DEVICE_ALWAYS = "device_always"
GATED = "gated"
STRATEGIES = (HOST_ONLY, DEVICE_ALWAYS, GATED)

DEFAULT_GRID = (1_000, 10_000, 20_000, 100_000, 500_000, 1_000_000, 3_000_000)
DEFAULT_REPEATS = 31
DEFAULT_MARGINS = (0.0, 5e-3, 10e-3)
_M64 = (1 << 64) - 1


@dataclass(frozen=True)
class WorkloadSpec:
    """Which sizes to run, how often, and with what mix (harness.py:82-117)."""

    n_grid: tuple = DEFAULT_GRID
    k: int = 100
    repeats: int = DEFAULT_REPEATS
    payload_bytes: int = DEFAULT_PAYLOAD_BYTES
    mix: Optional[tuple] = None
    seed: int = 0
    # tables' memory budget (store.generate_table); None: no cap (large-N key-only runs)
    memory_budget: Optional[int] = DEFAULT_MEMORY_BUDGET

    def __post_init__(self) -> None:
        grid = tuple(int(n) for n in self.n_grid)
        if not grid:
            raise ValueError("n_grid must be nonempty")
        if any(n < 1 for n in grid):
            raise ValueError("n_grid entries must be >= 1")
        if any(b <= a for a, b in zip(grid, grid[1:])):
            raise ValueError("n_grid must be strictly increasing")
        object.__setattr__(self, "n_grid", grid)
        if self.repeats < 1:
            raise ValueError("repeats must be >= 1")
        if self.payload_bytes < 1:
            raise ValueError("payload_bytes must be >= 1")
        if self.mix is not None:
            mix = tuple(float(w) for w in self.mix)
            if len(mix) != len(grid):
                raise ValueError("mix must have one weight per n_grid entry")
            if any(not math.isfinite(w) or w < 0 for w in mix):
                raise ValueError("mix weights must be finite and non-negative")
            total = math.fsum(mix)
            if total <= 0:
                raise ValueError("mix weights must not all be zero")
            object.__setattr__(self, "mix", tuple(w / total for w in mix))


@dataclass(frozen=True)
class LatencyStats:
    samples: tuple
    median: float
    p95: float
    p99: float
    mean: float


def _nearest_rank(ordered: Sequence[float], p: float) -> float:
    return ordered[max(1, math.ceil(p * len(ordered))) - 1]


def compute_stats(samples: Sequence[float]) -> LatencyStats:
    """Nearest-rank percentiles: index ceil(p*n), 1-based, on the sorted samples."""
    if len(samples) == 0:
        raise ValueError("compute_stats needs at least one sample")
    ordered = sorted(float(s) for s in samples)
    return LatencyStats(samples=tuple(float(s) for s in samples), median=_nearest_rank(ordered, 0.50),
                        p95=_nearest_rank(ordered, 0.95), p99=_nearest_rank(ordered, 0.99),
                        mean=math.fsum(ordered) / len(ordered))


@dataclass(frozen=True)
class StrategyRun:
    strategy: str
    per_n: dict
    offload_rate: float
    decisions: tuple = ()

    def all_samples(self) -> list:
        out: list = []
        for n in sorted(self.per_n):
            out.extend(self.per_n[n].samples)
        return out


def table_seed(spec_seed: int, n: int) -> int:
    return (spec_seed ^ mix64(n)) & _M64


class ScalingRow(NamedTuple):
    """One fig3 cell (harness.py:160-164)."""

    n: int
    op: str
    median_s: float
    p95_s: float


def run_scaling_baseline(spec: WorkloadSpec, backend: str = "modeled", cpu_model=None, device=None) -> list:
    """Cost per n of full_sort and topk -- the fig3 rows (harness.py:242-280).

    "modeled" reports the CPU cost model; any other backend wall-clock times the
    host primitives (one warmup run per cell). With `device` (a B200Device) the
    same cells are timed through the offload path as well, ops suffixed
    "@b200" (E2E wall time of device.full_sort / device.topk from host arrays),
    and each device answer is checked against the host primitive.
    """
    model = cpu_model if cpu_model is not None else DEFAULT_CPU_MODEL
    rows: list = []
    if backend == "modeled":
        for n in spec.n_grid:
            for op in (OP_FULL_SORT, OP_TOPK):
                v = estimate_cpu_cost(model, op, n, spec.k)
                rows.append(ScalingRow(n, op, v, v))
        return rows
    wall = lambda: time.perf_counter_ns() / 1e9  # noqa: E731
    for n in spec.n_grid:
        kv = random_key_vector(n, table_seed(spec.seed, n))
        cells = [(OP_FULL_SORT, lambda: host_full_sort(kv)), (OP_TOPK, lambda: host_topk(kv, spec.k))]
        if device is not None:
            sort_ref = host_full_sort(kv)
            topk_ref = host_topk(kv, spec.k).rows
            if not np.array_equal(device.full_sort(kv).payload, sort_ref):
                raise StrategyMismatchError(f"device full_sort differs from host_full_sort at n={n}")
            if not np.array_equal(device.topk(kv, spec.k).payload.rows, topk_ref):
                raise StrategyMismatchError(f"device topk differs from host_topk at n={n}")
            cells += [(OP_FULL_SORT + "@b200", lambda: device.full_sort(kv)),
                      (OP_TOPK + "@b200", lambda: device.topk(kv, spec.k))]
        for op, run in cells:
            run()
            samples = []
            for _ in range(spec.repeats):
                t0 = wall()
                run()
                samples.append(wall() - t0)
            st = compute_stats(samples)
            rows.append(ScalingRow(n, op, st.median, st.p95))
    return rows


def query_sizes(spec: WorkloadSpec) -> list:
    """The query sequence: grid x repeats, or seeded draws from the mix."""
    if spec.mix is None:
        return [n for n in spec.n_grid for _ in range(spec.repeats)]
    rng = np.random.Generator(np.random.PCG64(spec.seed & _M64))
    draws = rng.choice(np.asarray(spec.n_grid, dtype=np.int64), size=spec.repeats * len(spec.n_grid), p=spec.mix)
    return [int(x) for x in draws]


def _fingerprint(result) -> tuple:
    return (tuple(int(r) for r in result.row_ids), tuple(float(x) for x in result.keys))


def _run_one(table: ColumnTable, k: int, config: GateConfig, device, strategy: str):
    if strategy == GATED:
        result, decision, latency = execute_gated(table, OP_TOPK, k, config, device)
        return result, latency, decision
    result, latency = execute_path(table, OP_TOPK, k, config, device, HOST if strategy == HOST_ONLY else DEVICE)
    return result, latency, None


def run_strategy_comparison(spec: WorkloadSpec, config: GateConfig, device=None,
                            tables: Optional[dict] = None) -> tuple:
    """One identical Top-K query stream under host_only, device_always and gated.

    Answers are cross-checked per n before any latency is reported (a mismatch
    raises StrategyMismatchError). Non-modeled devices (b200) execute and
    wall-clock every query, discarding the first run per (n, strategy) cell.
    """
    if device is None:
        device = ModeledDevice(config.profile)
    modeled = getattr(device, "name", "") == "modeled"
    sizes = query_sizes(spec)
    tables = {} if tables is None else tables
    for n in spec.n_grid:
        if n not in tables:
            tables[n] = generate_table(n, spec.payload_bytes, seed=table_seed(spec.seed, n),
                                       memory_budget=spec.memory_budget)
    fingerprints: dict = {}
    first: dict = {}

    def check(strategy, n, result):
        fp = _fingerprint(result)
        if n not in fingerprints:
            fingerprints[n], first[n] = fp, strategy
        elif fingerprints[n] != fp:
            raise StrategyMismatchError(f"answers diverge at n={n}: strategy {strategy!r} disagrees with {first[n]!r}")

    runs = []
    for strategy in STRATEGIES:
        samples: dict = {n: [] for n in spec.n_grid}
        decisions: list = []
        offloaded = 0
        if modeled:
            cell = {}
            for n in spec.n_grid:
                result, latency, decision = _run_one(tables[n], spec.k, config, device, strategy)
                check(strategy, n, result)
                cell[n] = (latency, decision)
            for n in sizes:
                latency, decision = cell[n]
                samples[n].append(latency)
                if decision is not None:
                    decisions.append(decision)
                    offloaded += decision.path == DEVICE
        else:
            warmed: set = set()
            for n in sizes:
                if n not in warmed:
                    _run_one(tables[n], spec.k, config, device, strategy)
                    warmed.add(n)
                result, latency, decision = _run_one(tables[n], spec.k, config, device, strategy)
                check(strategy, n, result)
                samples[n].append(latency)
                if decision is not None:
                    decisions.append(decision)
                    offloaded += decision.path == DEVICE
        rate = {HOST_ONLY: 0.0, DEVICE_ALWAYS: 1.0}.get(strategy, offloaded / len(sizes) if sizes else 0.0)
        runs.append(StrategyRun(strategy, {n: compute_stats(s) for n, s in samples.items() if s}, rate,
                                tuple(decisions)))
    return tuple(runs)


class PayloadRow(NamedTuple):
    n: int
    mode: str
    bytes: int
    transfer_s: float


class TransferRow(NamedTuple):
    n: int
    mode: str
    h2d_bytes: int
    t_h2d: float
    t_kernel: float
    t_d2h: float
    t_post: float
    total_s: float


class E2eRow(NamedTuple):
    n: int
    mode: str
    e2e_s: float
    speedup_vs_full_row: float


@dataclass(frozen=True)
class PayloadComparison:
    payload_rows: list
    transfer_rows: list
    e2e_rows: list


def run_payload_comparison(spec: WorkloadSpec, device=None, profile=DEFAULT_MODELED_PROFILE) -> PayloadComparison:
    """Full-row vs key-only Top-K offload per n (the B axis of the gate sweep).
    Full-row E2E = t_h2d + t_kernel + t_d2h (payloads ride along); key-only E2E is
    the whole ledger (late materialization is t_post)."""
    device = device if device is not None else ModeledDevice(profile)
    payload_rows, transfer_rows, e2e_rows = [], [], []
    for n in spec.n_grid:
        kv = random_key_vector(n, table_seed(spec.seed, n))
        led = {}
        for mode in (FULL_ROW, KEY_ONLY):
            lg = device.topk(kv, spec.k, mode=mode, payload_bytes=spec.payload_bytes).ledger
            led[mode] = lg
            payload_rows.append(PayloadRow(n, mode, lg.h2d_bytes, lg.t_h2d))
            transfer_rows.append(TransferRow(n, mode, lg.h2d_bytes, lg.t_h2d, lg.t_kernel, lg.t_d2h, lg.t_post,
                                             lg.total))
        full = led[FULL_ROW]
        full_e2e = full.t_h2d + full.t_kernel + full.t_d2h
        key_e2e = led[KEY_ONLY].total
        e2e_rows.append(E2eRow(n, FULL_ROW, full_e2e, 1.0))
        e2e_rows.append(E2eRow(n, KEY_ONLY, key_e2e, full_e2e / key_e2e))
    return PayloadComparison(payload_rows, transfer_rows, e2e_rows)


def _timed_ledger(device, call):
    """A call's ledger for calibration. On a device that times its kernels with
    CUDA events (B200Device.time_kernels), t_kernel is that device time and the
    rest of the critical path is charged to the transfer phases (the ledger's
    wall-clock split puts only the kernel TAIL after the last upload into
    t_kernel, which does not grow with n: chunks are filtered / probed while
    later chunks upload). The phases still add up to the measured call time."""
    led = call().ledger
    timer = getattr(device, "last_kernel_seconds", None)
    k = timer() if timer is not None else None
    if not k:
        return led
    t_h2d = max(led.total - k - led.t_d2h - led.t_post, 0.0)
    return TransferLedger.build(led.h2d_bytes, led.d2h_bytes, t_h2d, k, led.t_d2h, led.t_post)


def calibrate_device_profile(device, ns: Sequence[int] = (100_000, 1_000_000, 4_000_000, 16_000_000), k: int = 100,
                             repeats: int = 3, seed: int = 0, probe_ns: Sequence[int] = ()):
    """Measured ledgers of `device` over an n grid -> DeviceProfile (the gate's C_gpu).

    For each n, the median-total ledger of `repeats` Top-K calls (after one
    warm-up) is kept; optional probe samples (build = probe = n/2, keys in
    [0, n)) calibrate kernel_rate_probe. A B200Device times its kernels with
    CUDA events during calibration, so kernel_rate_* are device rates.
    """
    timing = getattr(device, "time_kernels", None)
    if timing is not None:
        timing(True)
    try:
        return _calibrate(device, ns, k, repeats, seed, probe_ns)
    finally:
        if timing is not None:
            timing(False)


def _calibrate(device, ns, k, repeats, seed, probe_ns):
    samples = []
    for n in ns:
        kv = random_key_vector(n, table_seed(seed, n))
        device.topk(kv, k)
        leds = sorted((_timed_ledger(device, lambda: device.topk(kv, k)) for _ in range(repeats)),
                      key=lambda lg: lg.total)
        samples.append((n, leds[len(leds) // 2]))
    probe_samples = []
    for n in probe_ns:
        from .store import KeyVector

        rng = np.random.Generator(np.random.PCG64(table_seed(seed, n)))
        half = max(1, n // 2)
        b = KeyVector(rng.integers(0, n, half).astype(np.float64), np.arange(half, dtype=np.uint32))
        p = KeyVector(rng.integers(0, n, half).astype(np.float64), np.arange(half, dtype=np.uint32))
        device.probe(b, p)
        leds = sorted((_timed_ledger(device, lambda: device.probe(b, p)) for _ in range(repeats)),
                      key=lambda lg: lg.total)
        probe_samples.append((2 * half, leds[len(leds) // 2]))
    if len({n for n, _ in probe_samples}) >= 3:
        # Probes return tens of MB, so their ledgers pin both link bandwidths;
        # Top-K ledgers (a few hundred bytes back) then supply kernel_rate_topk.
        return calibrate_profile(probe_samples, op=OP_PROBE, probe_samples=samples)
    return calibrate_profile(samples, op=OP_TOPK, probe_samples=probe_samples)


__all__ = [
    "DEFAULT_GRID", "DEFAULT_MARGINS", "DEFAULT_REPEATS", "DEVICE_ALWAYS", "GATED", "HOST_ONLY", "STRATEGIES",
    "E2eRow", "LatencyStats", "PayloadComparison", "PayloadRow", "StrategyRun", "TransferRow", "WorkloadSpec",
    "calibrate_device_profile", "compute_stats", "query_sizes", "run_payload_comparison",
    "run_strategy_comparison", "table_seed",
]
