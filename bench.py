#!/usr/bin/env python
"""Benchmark of the B200 offload path (BASELINE.json metric, configs[1] by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload join_c2|topk_c1|topk_c3|join_c4]
    python bench.py --impl reference ...        # the reference's CPU algorithm (oracle port)

One step = one pass of the hot path over one batch of synthetic input:
  join_*  : hash-join build (all build keys) + probe (all probe keys), emitting
            (probe row, build row) pairs in reference order;
  topk_*  : Top-K over all keys.
N > 1 (torchrun, one process per GPU, NCCL) is STRONG scaling of the same global
workload: the probe side / the Top-K keys are split into contiguous shards
(sharded.shard_bounds) that keep their global row ids; the build side is
all-gathered (replicated table); Top-K candidates are all-gathered and merged.
`value`   = global Gkeys/s with inputs resident in HBM (device-timed CUDA
            events, max over ranks).
`e2e`     = the same metric through the public API (B200Device.probe/topk) from
            host numpy arrays: H2D + kernels + D2H + result objects; joins also
            report late materialization of the pairs (store.materialize_join).
`verify`  = the last timed step's output checked against the oracle (pairs in
            reference order / Top-K rows), outside the timed region.
Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Top-K/join-probe Gkeys/s (kernel & end-to-end); P95/P99 gated vs always-on vs CPU"

WORKLOADS = {
    # BASELINE.json configs[1] -- the default N=1 workload
    "join_c2": dict(kind="join", nb=1_000_000, np=10_000_000, seed=1,
                    desc="hash-join probe: build 1e6 / probe 1e7 uniform int64 keys in [0, 2e6) as f8, "
                         "emit (probe rowid, build rowid) pairs"),
    # BASELINE.json configs[0]
    "topk_c1": dict(kind="topk", n=1_000_000, k=100, seed=7,
                    desc="Top-K K=100 over N=1e6 uniform int64 keys in [0, 2^53) as f8 + rowids"),
    # BASELINE.json configs[2] (one K per run; --k to change)
    "topk_c3": dict(kind="topk", n=1_000_000_000, k=1000, seed=7,
                    desc="Top-K over N=1e9 uniform int64 keys in [0, 2^53) as f8 + rowids"),
    # BASELINE.json configs[3]
    "join_c4": dict(kind="join", nb=100_000_000, np=2_000_000_000, seed=1,
                    desc="hash-join probe: build 1e8 / probe 2e9 uniform int64 keys in [0, 2e8) as f8"),
}

VERIFY_WINDOW = 1 << 24  # probes per verified window of the large joins (prefix and suffix)


def _env_int(name: str, default: int) -> int:
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def bench_config(args, wl: dict) -> dict:
    """The workload description both arms print (identical by construction)."""
    cfg = {"workload": wl["desc"], "name": args.workload, "parallelism": f"dp{args.gpus}",
           "scaling": "strong: one global workload, sharded over the GPUs",
           "l2": "flushed between timed steps (256 MiB write outside the CUDA events)"}
    if wl["kind"] == "join":
        cfg.update(build_keys=wl["nb"], probe_keys=wl["np"], key_domain=2 * wl["nb"],
                   probe_row_ids="positions (arange)" if getattr(args, "probe_positions", False) else "u32 column")
    else:
        cfg.update(keys=wl["n"], k=wl["k"], dist=wl.get("dist", "uniform"),
                   row_ids="u32 column" if getattr(args, "row_column", False) else "positions (arange)")
    return cfg


def global_units(wl: dict) -> int:
    return wl["nb"] + wl["np"] if wl["kind"] == "join" else wl["n"]


# ---- synthetic data (the same global arrays on every rank) -------------------------

def join_data(wl: dict):
    """Build and probe columns: uniform integers in [0, 2*nb) as f8, row ids = positions."""
    nb, np_ = wl["nb"], wl["np"]
    rng = np.random.Generator(np.random.PCG64(wl["seed"]))
    bk = rng.integers(0, 2 * nb, size=nb).astype(np.float64)
    pk = rng.integers(0, 2 * nb, size=np_).astype(np.float64)
    return bk, np.arange(nb, dtype=np.uint32), pk, np.arange(np_, dtype=np.uint32)


def topk_data(wl: dict):
    """Uniform keys (random_keys, store.py:165-171) or the SURVEY 8(d) Zipf variants:
    r = PCG64(11).zipf(1.2, N) clipped to 2^53-1; "zipf_hi" key = (2^53-1) - r (the
    most frequent rank is the largest key: K reduces to the smallest row ids among
    the ties), "zipf_lo" key = r (the heavy tail sets the threshold)."""
    n = wl["n"]
    dist = wl.get("dist", "uniform")
    if dist == "uniform":
        rng = np.random.Generator(np.random.PCG64(wl["seed"]))
        keys = rng.integers(0, 2**53, size=n, dtype=np.int64).astype(np.float64)
    else:
        rng = np.random.Generator(np.random.PCG64(11))
        r = np.minimum(rng.zipf(1.2, n), 2**53 - 1).astype(np.float64)
        keys = (2.0**53 - 1) - r if dist == "zipf_hi" else r
    return keys, np.arange(n, dtype=np.uint32)


# ---- clocks (NVML, sampled during the timed region) --------------------------------

_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
            0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    """Samples the SM clock and the clock-event reasons in a background thread
    (every `period_s`, as fast as NVML answers when 0) while the timed region runs."""

    def __init__(self, device_index: int, period_s: float = 0.0005):
        self.samples: list[tuple[int, int]] = []
        self.period = period_s
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = int(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:  # NVML unavailable: report null clocks
            self._nv = None

    def _run(self):
        nv = self._nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append((int(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)),
                                     int(get_reasons(self._h))))
            except Exception:
                pass
            if self.period:
                time.sleep(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
            while not self.samples and self._t.is_alive():  # at least one sample before timing starts
                time.sleep(0.0002)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        mhz = [s[0] for s in self.samples]
        bits = 0
        for _, r in self.samples:
            bits |= r
        reasons = [name for b, name in _REASONS.items() if bits & b and name != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(mhz)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples)}


# ---- reference arm / CPU baseline ------------------------------------------------------

def cpu_reference_steps(wl: dict, steps: int, warmup: int, data, threads: int) -> tuple[float, str]:
    """Times the reference's CPU algorithm (oracle port of ProxyDevice: serial
    KeyHashTable build + chunk-parallel probe / chunk top-k + merge)."""
    from oracle import oracle

    oracle.build()
    times = []
    if wl["kind"] == "join":
        bk, br, pk, pr = data
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            t = oracle.Table(bk, br)
            t.probe(pk, pr, workers=threads)
            dt = time.perf_counter() - t0
            if i >= warmup:
                times.append(dt)
        units = len(bk) + len(pk)
        sample = (f"serial build of {len(bk)} + {threads}-thread probe of {len(pk)} "
                  f"(oracle port of ProxyDevice.probe, device.py:382-436)")
    else:
        keys, rows = data
        k = wl["k"]
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            oracle.proxy_topk(keys, rows, k, threads)
            dt = time.perf_counter() - t0
            if i >= warmup:
                times.append(dt)
        units = len(keys)
        sample = (f"{threads}-thread chunk top-{k} + merge over {len(keys)} keys "
                  f"(oracle port of ProxyDevice.topk, device.py:329-380)")
    return units / statistics.mean(times) / 1e9, sample


def bounded_sample(wl: dict, data):
    """The CPU legs run the full C1/C2 workloads; the 1e9-scale configs are sampled
    (1e8 Top-K keys; build 1e7 / probe 1e8) so a run ends within minutes."""
    if wl["kind"] == "topk" and wl["n"] > 100_000_000:
        return (data[0][:100_000_000], data[1][:100_000_000]), True
    if wl["kind"] == "join" and wl["np"] > 100_000_000:
        return (data[0][:10_000_000], data[1][:10_000_000], data[2][:100_000_000], data[3][:100_000_000]), True
    return data, False


def run_reference(args, wl) -> None:
    rank = _env_int("RANK", 0)
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    data = join_data(wl) if wl["kind"] == "join" else topk_data(wl)
    data, sampled = bounded_sample(wl, data)
    value, sample = cpu_reference_steps(wl, args.steps, args.warmup, data, threads)
    if sampled:
        sample += "; sampled workload, ms_per_step extrapolated to the full workload at the sampled rate"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gkeys/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": global_units(wl) / (value * 1e9) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, wl),
        "cpu_baseline": {"value": value, "unit": "Gkeys/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "Gkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- verification of the timed outputs (outside the timed region) ----------------------

def verify_join(bk, br, pk_s, pr_s, got_p: np.ndarray, got_b: np.ndarray, m: int, threads: int) -> dict:
    """This rank's pairs vs the oracle's KeyHashTable probe of this rank's probe
    shard (reference order). Shards up to 2^26 probes are checked whole; larger
    ones on a prefix and a suffix window (aligned by pair counts)."""
    from oracle import oracle

    table = oracle.Table(bk, br)
    n = len(pk_s)
    if n <= 1 << 26:
        wp, wb = table.probe(pk_s, pr_s, workers=threads)
        ok = m == len(wp) and np.array_equal(got_p, wp) and np.array_equal(got_b, wb)
        return {"ok": bool(ok), "checked": f"all {m} pairs of {n} probes vs oracle (reference order)"}
    w = VERIFY_WINDOW
    hp, hb = table.probe(pk_s[:w], pr_s[:w], workers=threads)
    tp, tb = table.probe(pk_s[-w:], pr_s[-w:], workers=threads)
    ok = (len(hp) + len(tp) <= m and np.array_equal(got_p[:len(hp)], hp) and np.array_equal(got_b[:len(hb)], hb)
          and np.array_equal(got_p[m - len(tp):m], tp) and np.array_equal(got_b[m - len(tb):m], tb))
    return {"ok": bool(ok), "checked": f"pairs of the first and last {w} of {n} probes vs oracle "
                                       f"({len(hp)} + {len(tp)} of {m} pairs, reference order)"}


def verify_topk(keys, rows, k: int, got: np.ndarray, threads: int) -> dict:
    from oracle import oracle

    want = oracle.proxy_topk(keys, rows, k, threads)
    return {"ok": bool(np.array_equal(got, want)), "checked": f"all {len(want)} rows vs oracle over {len(keys)} keys"}


# ---- B200 arm --------------------------------------------------------------------------

def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "fallback": True}


def _traffic(workload: str):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        return json.loads(p.read_text()).get(workload)
    return None


def run_b200(args, wl) -> None:
    import torch
    import torch.distributed as dist

    from paper_2601_19911_b200 import B200Device, KeyVector, _native, resident, sharded
    from paper_2601_19911_b200.store import ColumnTable, materialize_join

    rank, world, local = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1), _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _native.load()
    device = B200Device(device=local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()
    threads = os.cpu_count() or 1

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: int) -> int:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        return int(t.item())

    units = global_units(wl)
    if wl["kind"] == "join":
        bk, br, pk, pr = join_data(wl)
        blo, bhi = sharded.shard_bounds(len(bk), world, rank)
        lo, hi = sharded.shard_bounds(len(pk), world, rank)
        pk_s, pr_s = pk[lo:hi], pr[lo:hi]  # this rank's probe shard keeps its global row ids
        t_bk = torch.from_numpy(bk[blo:bhi]).to(dev)
        t_br = torch.from_numpy(br[blo:bhi].view(np.int32)).to(dev)
        t_pk = torch.from_numpy(pk_s).to(dev)
        # the probe row ids are the positions (extract_keys's arange); by default they
        # travel as a u32 column (12 B per probe); --probe-positions passes
        # the shard's first row id instead (golp_join_probe_device_positions, 8 B per probe)
        t_pr = int(lo) if args.probe_positions else torch.from_numpy(pr_s.view(np.int32)).to(dev)
        # size the pair buffers once (first call), then reuse them every step
        full_bk = torch.cat(sharded._all_gather_ragged(t_bk)) if world > 1 else t_bk
        full_br = torch.cat(sharded._all_gather_ragged(t_br)) if world > 1 else t_br
        op0, _ = resident.join(full_bk, full_br, t_pk, t_pr)
        cap = max(int(op0.numel()), 1)
        out_p = torch.empty(cap, dtype=torch.int32, device=dev)
        out_b = torch.empty(cap, dtype=torch.int32, device=dev)
        del op0, full_bk, full_br
        m_dev = torch.zeros(1, dtype=torch.int64, device=dev)

        def step_build():
            if world > 1:
                fbk = torch.cat(sharded._all_gather_ragged(t_bk))
                fbr = torch.cat(sharded._all_gather_ragged(t_br))
            else:
                fbk, fbr = t_bk, t_br
            resident.join_build(fbk, fbr)

        def step_probe():
            resident.join_probe_async(t_pk, t_pr, out_p, out_b, m_dev)
            return m_dev

        def step():
            # build + probe fully enqueued; the match count stays on the device
            # (read after the step's end event, checked against the capacity)
            step_build()
            return step_probe()

        local_units = len(bk) + len(pk_s)
    else:
        keys, rows = topk_data(wl)
        lo, hi = sharded.shard_bounds(len(keys), world, rank)
        t_k = torch.from_numpy(keys[lo:hi]).to(dev)
        # the row ids are the positions (extract_keys's arange): by default the step
        # passes the shard's first row id instead of a row column (no row loads for
        # threshold ties); --row-column keeps the u32 column in HBM
        t_r = torch.from_numpy(rows[lo:hi].view(np.int32)).to(dev) if args.row_column else int(lo)
        k = wl["k"]

        def step():
            return sharded.topk(t_k, t_r, k)

        local_units = hi - lo

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # One CUDA graph per step where the step is a pure enqueue (no host round
    # trip): the fused C1-sized Top-K, and the join step as two graphs (build,
    # probe) with a CUDA event on the stream between them, so the probe phase is
    # timed by that event and the step's end event -- no event nodes inside the
    # graphs (each costs ~2.7 us per step). Other paths time their kernel groups
    # with the library's events on the launch stream.
    split = wl["kind"] == "join" and world == 1 and not args.no_graph
    capturable = wl["kind"] == "join" or (local_units <= 2_000_000 and wl["k"] <= 4096)
    # the C1-sized Top-K graph is one fused kernel: time the whole replay with the
    # step's own events (no event nodes inside the graph)
    whole = wl["kind"] != "join" and world == 1 and capturable and not args.no_graph
    resident.set_profiling(not (split or whole))
    graph, graph_launches = None, 0
    if world == 1 and capturable and not args.no_graph:
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            for _ in range(2):
                step()
        stream.wait_stream(side)
        torch.cuda.synchronize()
        l0 = _native.launch_count()
        if split:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step_build()
            graph_p = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph_p):
                graph_out = step_probe()
        else:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                graph_out = step()
        graph_launches = _native.launch_count() - l0
        torch.cuda.synchronize()
        graph.replay()
        if split:
            graph_p.replay()
        torch.cuda.synchronize()
    kern_ms, step_ms = [], []
    fused = False
    out = None
    barrier()
    torch.cuda.synchronize()
    launches0 = _native.launch_count()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            em = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if graph is not None:
                graph.replay()
                if split:
                    em.record(stream)
                    graph_p.replay()
                out = graph_out
            else:
                out = step()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            if wl["kind"] == "join":
                assert int(out.item()) <= cap, "pair buffers too small for the timed step"
            kt = _native.kernel_times()
            if split:
                kern_ms.append(em.elapsed_time(e1))
            elif whole:
                kern_ms.append(step_ms[-1])
                fused = True
            elif wl["kind"] == "join":
                kern_ms.append(kt["join_probe_ms"])
            elif kt["topk_filter_ms"] > 0:
                kern_ms.append(kt["topk_filter_ms"])
            else:  # fused small Top-K: one kernel covers threshold + filter + select
                kern_ms.append(kt["topk_select_ms"])
                fused = True
    torch.cuda.synchronize()
    barrier()
    launches = _native.launch_count() - launches0 + graph_launches * args.steps
    resident.set_profiling(False)
    ms = max_over_ranks(statistics.mean(step_ms))
    value = units / (ms / 1e3) / 1e9

    # the last timed step's output vs the oracle (each rank checks its shard)
    if wl["kind"] == "join":
        matches = int(out.item())
        got_p = out_p[:matches].cpu().numpy().view(np.uint32)
        got_b = out_b[:matches].cpu().numpy().view(np.uint32)
        verify = verify_join(bk, br, pk_s, pr_s, got_p, got_b, matches, threads) if not args.no_verify else None
        matches_total = sum_over_ranks(matches)
    else:
        got = out.cpu().numpy().view(np.uint32)
        verify = verify_topk(keys, rows, k, got, threads) if (rank == 0 and not args.no_verify) else None
        matches_total = None
    if wl["kind"] == "join" and verify is not None and world > 1:  # every rank checked its shard
        oks = [None] * world
        dist.all_gather_object(oks, verify["ok"])
        verify["ok"] = all(oks)
        verify["checked"] += f" (each of {world} ranks)"
    if verify is not None and not verify["ok"]:
        raise SystemExit(f"bench output does not match the oracle: {verify}")

    # roofline of the dominant kernel (per launch, algorithmic bytes; this rank)
    peaks = _peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    kms = statistics.mean(kern_ms)
    if wl["kind"] == "join":
        table_bytes = int(kt["join_capacity"]) * 16
        l2 = torch.cuda.get_device_properties(dev).L2_cache_size
        # 8-byte key (+ 4-byte row id when a row column is read; positions are computed)
        per_probe = (8 if args.probe_positions else 12) + (32 if table_bytes > l2 else 0)
        alg_bytes = per_probe * len(pk_s) + 8 * matches
        kernel = "join_probe (join_match_kernel + join_emit_kernel)"
    else:
        alg_bytes = 8 * local_units
        kernel = ("topk_fused_kernel (whole graph replay, step events)" if whole
                  else "topk_fused_kernel" if fused else "topk_filter_kernel")
    achieved = alg_bytes / (kms / 1e3) / 1e9

    # end to end through the public API from host numpy arrays. Default device:
    # reused input columns get page-locked after their 2nd use (PinCache), results
    # land in the pinned result arena; a second device with pinning off gives the
    # staged (pageable-copy, first-touch) number for the same calls.
    big = units > 200_000_000  # 1e9-scale workloads: bounded E2E sample (12 GB per call)
    e2e_steps, e2e_warm = (min(args.steps, 2), 2) if big else (args.steps, args.warmup)
    if wl["kind"] == "join":
        kv_b, kv_p = KeyVector(bk, br), KeyVector(pk_s, pr_s)
        h2d_ref = 12 * (len(bk) + len(pk_s))
    else:
        kv = KeyVector(keys[lo:hi], rows[lo:hi])
        h2d_ref = 12 * (hi - lo)

    def merge_topk(local_rows: np.ndarray) -> np.ndarray:
        """Global top-K from every rank's local top-K (rank 0 merges on the host by
        key desc, row asc -- host_topk's order, host.py:141)."""
        if world == 1:
            return local_rows
        parts = [None] * world
        dist.all_gather_object(parts, local_rows)
        cand = np.concatenate(parts)
        ck = keys[cand]  # row ids are global positions here
        order = np.lexsort((cand, -(ck + 0.0)))
        return cand[order[:k]]

    def e2e_run(dev_):
        ts = []
        res_ = None
        for i in range(e2e_warm + e2e_steps):
            barrier()
            t0 = time.perf_counter()
            if wl["kind"] == "join":
                res_ = dev_.probe(kv_b, kv_p)
            else:
                res_ = dev_.topk(kv, wl["k"])
                merge_topk(res_.payload.rows)
            dt = time.perf_counter() - t0
            if i >= e2e_warm:
                ts.append(dt)
        return statistics.mean(ts), res_

    staged_s, _ = e2e_run(B200Device(device=local, pin_inputs=False)) if not big else (float("nan"), None)
    rows_copied_s, _ = e2e_run(B200Device(device=local, dense_rows=False))
    e2e_mean, res = e2e_run(device)
    # bytes the copy engines actually moved in the last timed call: the key
    # columns, plus the row-id columns unless they are a dense run
    h2d, d2h = _native.last_transfer()
    e2e_s = max_over_ranks(e2e_mean)
    e2e_value = units / e2e_s / 1e9
    staged_s = max_over_ranks(staged_s)
    rows_copied_s = max_over_ranks(rows_copied_s)
    e2e = {"value": e2e_value, "unit": "Gkeys/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": e2e_s * 1e3,
           "input_pinning": "input columns page-locked in place after their 2nd use (PinCache); results DMA "
                            "into the pinned result arena",
           "row_ids": "dense row-id columns (arange, as extract_keys makes them) are verified on the host inside "
                      "the timed call and regenerated on the device, not copied",
           "h2d_bytes_reference_accounting": h2d_ref,
           "rows_copied_value": units / rows_copied_s / 1e9, "rows_copied_ms_per_step": rows_copied_s * 1e3,
           "staged_value": None if math.isnan(staged_s) else units / staged_s / 1e9,
           "staged_ms_per_step": None if math.isnan(staged_s) else staged_s * 1e3,
           "last_ledger_ms": {f: getattr(res.ledger, f) * 1e3 for f in ("t_h2d", "t_kernel", "t_d2h", "t_post")}}
    if wl["kind"] == "join" and not big:
        # late materialization of the pairs (store.materialize_join):
        # keys + 188-byte payloads of both sides gathered in pair order
        pb = 188
        bt = ColumnTable(bk, np.full((len(bk), pb), 7, dtype=np.uint8), 0)
        pt = ColumnTable(pk, np.full((len(pk), pb), 9, dtype=np.uint8), 1)
        mts = []
        for _ in range(3):
            t0 = time.perf_counter()
            mj = materialize_join(bt, pt, res.payload)
            mts.append(time.perf_counter() - t0)
        mat_s = max_over_ranks(min(mts))
        assert len(mj) == res.payload.match_count
        e2e.update(materialize_ms=mat_s * 1e3, materialize_payload_bytes=pb,
                   with_materialize_value=units / (e2e_s + mat_s) / 1e9,
                   with_materialize_ms_per_step=(e2e_s + mat_s) * 1e3)
        del bt, pt, mj

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        data = (bk, br, pk, pr) if wl["kind"] == "join" else (keys, rows)
        data, _ = bounded_sample(wl, data)
        cv, sample = cpu_reference_steps(wl, 3, 1, data, threads)
        cpu = {"value": cv, "unit": "Gkeys/s", "cores": threads, "kind": "port", "sample": sample}

    device.close()
    if rank == 0:
        details = {"global_units_per_step": units, "units_per_rank": local_units,
                   "launch": ("cuda-graph replays per step: build graph, stream event, probe graph" if split
                              else "cuda-graph replay per step" if graph is not None else "eager launches")}
        if matches_total is not None:
            details["matches"] = matches_total
        line = {
            "metric": METRIC, "value": value, "unit": "Gkeys/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": bench_config(args, wl),
            "details": details, "e2e": e2e, "verify": verify,
            "roofline": {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _traffic(args.workload),
                         "frac_of_nominal_8tbs": achieved / 8000.0,
                         "algorithmic_bytes_per_launch": alg_bytes, "kernel_ms": kms,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "fallback" not in peaks else "fallback"},
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        if wl["kind"] == "join":
            line["roofline"]["build_ms"] = statistics.mean(step_ms) - kms  # step minus probe phase
            # The probe is bound by random table lookups, not by HBM bytes: one
            # 32-byte slot-pair read per probe. Its ceiling is the measured rate of
            # random 32-B loads from an L2-resident table (tools/probe_ladder.cu
            # rung 1: ~207-244 G/s, the L1TEX one-wavefront-per-clock limit); tables
            # larger than L2 are capped by DRAM-random reads (~40 G/s measured).
            # (the radix-partitioned path makes C4's lookups L2 lookups, so it is
            # held to the L2 ceiling too).
            table_in_l2 = table_bytes <= l2
            partitioned = int(kt["join_slices"]) > 1
            ceiling = LOOKUP_CEILING_L2 if (table_in_l2 or partitioned) else LOOKUP_CEILING_DRAM
            lookups = len(pk_s) / (kms / 1e3) / 1e9
            where = "L2-resident table" if table_in_l2 else ("table > L2, slice-partitioned" if partitioned
                                                             else "table > L2")
            line["roofline"]["lookup"] = {
                "bound": f"random 32-B table lookups ({where})",
                "achieved": lookups, "peak": ceiling, "unit": "Glookups/s", "frac": lookups / ceiling,
                "peak_source": "tools/probe_ladder.cu, tools/microbench.cu (B200)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


LOOKUP_CEILING_L2 = 244.0    # G random 32-B lookups/s, L2-resident table
LOOKUP_CEILING_DRAM = 40.0   # G random 32-B lookups/s, table in HBM


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="join_c2")
    ap.add_argument("--k", type=int, default=None, help="override K for topk workloads")
    ap.add_argument("--dist", choices=("uniform", "zipf_hi", "zipf_lo"), default="uniform",
                    help="key distribution of the Top-K workloads")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the oracle check of the timed output")
    ap.add_argument("--no-graph", action="store_true", help="launch every resident step eagerly")
    ap.add_argument("--row-column", action="store_true",
                    help="Top-K: pass the row-id column instead of the positions it holds")
    ap.add_argument("--probe-positions", action="store_true",
                    help="joins: pass the probe side's row ids as positions instead of a u32 column")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    wl = dict(WORKLOADS[args.workload])
    if args.k is not None:
        wl["k"] = args.k
    if args.dist != "uniform":
        if wl["kind"] != "topk":
            raise SystemExit("--dist applies to the Top-K workloads")
        wl["dist"] = args.dist
        wl["desc"] = wl["desc"].replace("uniform", args.dist.replace("_", "-") + " (SURVEY 8(d))")
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_b200(args, wl)


if __name__ == "__main__":
    main()
