"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (needs /root/reference, which does not travel
to the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/{topk,probe,table,gate}.npz. Inputs and the reference's own
outputs are stored, so the oracle (oracle/oracle.c) and the B200 path are
checked against what `golp` actually returns, not against a restatement.
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _ref():
    sys.path.insert(0, str(REF))
    import golp  # noqa: F401  (the reference, imported read-only)
    from golp import device, gate, harness, host, store
    return golp, device, gate, harness, host, store


class Packer:
    """Ragged list of cases -> flat arrays + offsets (npz friendly)."""

    def __init__(self):
        self.cols: dict[str, list[np.ndarray]] = {}
        self.scalars: dict[str, list] = {}

    def add(self, arrays: dict[str, np.ndarray], **scalars):
        for k, v in arrays.items():
            self.cols.setdefault(k, []).append(np.asarray(v))
        for k, v in scalars.items():
            self.scalars.setdefault(k, []).append(v)

    def save(self, path: Path):
        out = {}
        for k, parts in self.cols.items():
            out[k] = np.concatenate(parts) if parts else np.empty(0)
            out[k + "_off"] = np.cumsum([0] + [len(p) for p in parts]).astype(np.int64)
        for k, vals in self.scalars.items():
            out[k] = np.asarray(vals)
        np.savez_compressed(path, **out)


def topk_cases(golp, host, store):
    pk = Packer()

    def add(keys, rows, k, tag):
        kv = store.KeyVector(keys=np.asarray(keys, dtype=np.float64), rows=np.asarray(rows, dtype=np.uint32))
        got = host.host_topk(kv, k).rows
        pk.add({"keys": kv.keys, "rows": kv.rows, "expect": got}, k=k, tag=tag)

    # hand cases (pkg/tests/test_host.py:51-71) and SURVEY 8(c) extra vectors
    add([5, 1, 9, 3], range(4), 2, "hand")
    add([4.0, 4.0, -1.0, 7.0], range(4), 10, "k_ge_n")
    add([7, 7, 7, 7], [9, 2, 5, 1], 2, "ties")
    add([0.0, -0.0, 0.0, -1.0], [5, 2, 9, 1], 2, "neg_zero")
    big = np.array([2**53, 2**53 + 1, 2**53 - 1], dtype=np.int64).astype(np.float64)
    add(big, [7, 3, 0], 1, "beyond_2p53")
    add([-3.5, -1e300, 1e300, -0.0, 0.0, 5e-324, -5e-324], [6, 5, 4, 3, 2, 1, 0], 7, "extremes")
    add([1.0], [0], 1, "single")
    # crit-1 style random instances (pkg/tests/test_acceptance.py:74-91), smaller n
    rng = np.random.default_rng(20260816)
    for i in range(120):
        n = int(10 ** rng.uniform(1, 3.7))
        k = int(rng.choice([1, 10, 100, max(1, n)]))
        if i % 3 == 0:
            keys = rng.integers(0, max(2, n // 8), size=n).astype(np.float64)
        else:
            keys = rng.standard_normal(n)
        add(keys, rng.permutation(n), k, "crit1")
    # heavy ties in tiny domains (test_host.py:97-105 shape)
    rng = np.random.default_rng(97)
    for _ in range(40):
        n = int(rng.integers(1, 60))
        keys = rng.integers(-5, 6, size=n).astype(np.float64)
        keys[rng.random(n) < 0.2] = -0.0
        add(keys, rng.permutation(n), int(rng.integers(1, 65)), "heavy_ties")
    # many ties straddling the K boundary at larger n, both row orders
    rng = np.random.default_rng(5)
    for k in (1, 37, 500, 4096, 5000):
        keys = rng.integers(0, 16, size=20_000).astype(np.float64)
        add(keys, rng.permutation(20_000), k, "boundary_ties")
        add(keys, np.arange(20_000), k, "boundary_ties_arange")
    pk.save(OUT / "topk.npz")
    # generator parity + a larger known answer: random_key_vector(100000, 3), k=100
    kv = store.random_key_vector(100_000, 3)
    ans = host.host_topk(kv, 100).rows
    np.savez_compressed(OUT / "topk_large.npz", n=100_000, seed=3, k=100, expect=ans,
                        key_sum=np.float64(kv.keys.sum()), key_head=kv.keys[:16])


def probe_cases(golp, host, store):
    pk = Packer()

    def add(bk, br, pkk, pr, tag):
        b = store.KeyVector(keys=np.asarray(bk, dtype=np.float64), rows=np.asarray(br, dtype=np.uint32))
        p = store.KeyVector(keys=np.asarray(pkk, dtype=np.float64), rows=np.asarray(pr, dtype=np.uint32))
        res = host.host_hash_probe(host.host_hash_build(b), p)
        pk.add({"bkeys": b.keys, "brows": b.rows, "pkeys": p.keys, "prows": p.rows,
                "exp_p": res.probe_rows, "exp_b": res.build_rows}, tag=tag)

    add([1, 2, 3], range(3), [2, 2, 5], range(3), "hand")
    add([], [], [1, 2], range(2), "empty_build")
    add([1, 2], range(2), [], [], "empty_probe")
    add([7, 7], [0, 1], [7], [5], "dup_build")
    add([0.0], [0], [-0.0], [0], "neg_zero")
    add([-3.5, 2.0, -3.5], [0, 1, 2], [-3.5], [9], "negative")
    add([4, 4, 4], [30, 10, 20], [4, 1, 4], [8, 9, 7], "insertion_order")
    add([1.0, 2.0], [0, 1], [5.0, 6.0], [0, 1], "no_match")
    rng = np.random.default_rng(21)
    for _ in range(60):  # pkg/tests/test_host.py:128-138 shape
        nb, npr = int(rng.integers(1, 1000)), int(rng.integers(1, 1000))
        bk = rng.integers(0, 50, size=nb).astype(np.float64)
        pkk = rng.integers(0, 50, size=npr).astype(np.float64)
        add(bk, rng.permutation(nb), pkk, rng.permutation(npr), "small_domain")
    rng = np.random.default_rng(20260816)
    for _ in range(60):  # crit-1 probe shape (test_acceptance.py:93-105)
        nb = int(10 ** rng.uniform(1, 3.5))
        npr = int(10 ** rng.uniform(1, 3.5))
        domain = max(4, (nb + npr) // 3)
        bk = rng.integers(0, domain, size=nb).astype(np.float64)
        pkk = rng.integers(0, domain, size=npr).astype(np.float64)
        add(bk, rng.permutation(nb), pkk, rng.permutation(npr), "crit1")
    rng = np.random.default_rng(44)
    for _ in range(6):  # large duplicate groups (> 32 and > a warp) in build order
        nb = int(rng.integers(100, 3000))
        bk = rng.integers(0, 3, size=nb).astype(np.float64)
        pkk = rng.integers(0, 4, size=50).astype(np.float64)
        add(bk, rng.permutation(nb), pkk, rng.permutation(50), "big_groups")
    pk.save(OUT / "probe.npz")


def table_layout(golp, host, store):
    rng = np.random.default_rng(8)
    keys = rng.integers(0, 40, size=300).astype(np.float64)
    keys[::7] = -0.0
    rows = rng.permutation(300).astype(np.uint32)
    t = host.host_hash_build(store.KeyVector(keys=keys, rows=rows))
    vals = rng.integers(0, 2**63, size=64, dtype=np.int64).astype(np.uint64) * np.uint64(2)
    mixed = np.array([host.mix64(int(v)) for v in vals.tolist()], dtype=np.uint64)
    np.savez_compressed(OUT / "table.npz", keys=keys, rows=rows, capacity=t.capacity, slot_bits=t.slot_bits,
                        slot_rows=t.slot_rows, mix_in=vals, mix_out=mixed)


def gate_cases(golp, device, gate, harness):
    """decide()/estimate/calibration numbers of the reference, for the Python layer."""
    out = {"decide": [], "estimate": [], "calibrate_profile": None, "calibrate_cpu": None, "stats": []}
    cfgs = {
        "default": gate.GateConfig(),
        "margin5ms": gate.GateConfig(margin_s=5e-3),
        "guard20k": gate.GateConfig(min_n_guard=20_000),
        "full_row": gate.GateConfig(mode=device.FULL_ROW),
    }
    for name, cfg in cfgs.items():
        for op in (device.OP_TOPK, device.OP_PROBE):
            for n in (0, 1_000, 10_000, 20_000, 100_000, 500_000, 1_000_000, 3_000_000, 10**9):
                for k in (1, 100, 100_000):
                    for build_n in ((0,) if op == device.OP_TOPK else (0, 1_000_000)):
                        pb = 188 if cfg.mode == device.FULL_ROW else None
                        d = gate.decide(cfg, op, n, k, pb, build_n)
                        out["decide"].append([name, op, n, k, build_n, d.path, d.c_cpu_est, d.c_gpu_est, d.gain,
                                              d.guard_triggered])
    for op in (device.OP_TOPK, device.OP_PROBE):
        for n in (0, 1, 99, 20_000, 3_000_000):
            for mode, pb in ((device.KEY_ONLY, None), (device.FULL_ROW, 188)):
                e = device.estimate_device_cost(op, n, 100, mode, pb)
                out["estimate"].append([op, n, mode, list(e)])
    rng = np.random.default_rng(3)
    samples = []
    for n in (1_000, 10_000, 100_000, 1_000_000, 5_000_000):
        led = device.TransferLedger.build(12 * n, 400, 12 * n / 40e9 * (1 + 0.05 * rng.standard_normal()),
                                          20e-6 + n * 1e-12 * (1 + 0.05 * rng.standard_normal()), 400 / 20e9,
                                          100 * 5e-9)
        samples.append((n, led))
    prof = device.calibrate_profile(samples)
    out["calibrate_profile"] = {"samples": [[n, list(led.__dict__.values())] for n, led in samples],
                                "profile": prof.to_json_dict()}
    cpu_samples = [("topk", n, 100, 1.2e-10 * n * math.log2(n) * (1 + 0.01 * i) + 5e-6)
                   for i, n in enumerate((10_000, 100_000, 1_000_000))]
    cpu_samples += [("probe", n, 2, 5e-10 * n * 2 * (1 + 0.01 * i) + 5e-6)
                    for i, n in enumerate((10_000, 100_000, 1_000_000))]
    out["calibrate_cpu"] = {"samples": cpu_samples,
                            "model": gate.calibrate_cpu_model(cpu_samples).to_json_dict()}
    for seq in ([1.0], [3.0, 1.0, 2.0], list(np.linspace(0, 1, 101)), [5, 5, 1, 9, 2, 2, 7]):
        s = harness.compute_stats(seq)
        out["stats"].append([list(map(float, seq)), s.median, s.p95, s.p99, s.mean])
    spec = harness.WorkloadSpec(n_grid=(1_000, 100_000, 10**9), k=100, repeats=3)
    out["scaling_modeled"] = [list(r) for r in harness.run_scaling_baseline(spec, backend="modeled")]
    (OUT / "gate.json").write_text(json.dumps(out, indent=0))


def full_sort_cases(golp, host, store):
    """host_full_sort (pkg/src/golp/host.py:127-130) known answers."""
    pk = Packer()

    def add(keys, rows, tag):
        kv = store.KeyVector(keys=np.asarray(keys, dtype=np.float64), rows=np.asarray(rows, dtype=np.uint32))
        pk.add({"keys": kv.keys, "rows": kv.rows, "expect": host.host_full_sort(kv)}, tag=tag)

    add([5, 1, 9, 3], range(4), "hand")
    add([7, 7, 7, 7], [9, 2, 5, 1], "ties")
    add([0.0, -0.0, 0.0, -1.0], [5, 2, 9, 1], "neg_zero")
    big = np.array([2**53, 2**53 + 1, 2**53 - 1], dtype=np.int64).astype(np.float64)
    add(big, [7, 3, 0], "beyond_2p53")
    add([-3.5, -1e300, 1e300, -0.0, 0.0, 5e-324, -5e-324], [6, 5, 4, 3, 2, 1, 0], "extremes")
    add([1.0], [0], "single")
    rng = np.random.default_rng(127)
    for i in range(30):
        n = int(10 ** rng.uniform(1, 4.3))
        if i % 3 == 0:
            keys = rng.integers(-4, 5, size=n).astype(np.float64)
            keys[rng.random(n) < 0.2] = -0.0
        elif i % 3 == 1:
            keys = rng.standard_normal(n)
        else:
            keys = rng.integers(0, 2**53, size=n, dtype=np.int64).astype(np.float64)
        rows = np.arange(n) if i % 2 else rng.permutation(n)
        add(keys, rows, "random")
    pk.save(OUT / "full_sort.npz")


GENERATORS = ("topk", "probe", "table", "gate", "full_sort")


def main(which=GENERATORS):
    golp, device, gate, harness, host, store = _ref()
    if "topk" in which:
        topk_cases(golp, host, store)
    if "probe" in which:
        probe_cases(golp, host, store)
    if "table" in which:
        table_layout(golp, host, store)
    if "gate" in which:
        gate_cases(golp, device, gate, harness)
    if "full_sort" in which:
        full_sort_cases(golp, host, store)
    for p in sorted(OUT.glob("*.npz")) + [OUT / "gate.json"]:
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main(tuple(sys.argv[1:]) or GENERATORS)
