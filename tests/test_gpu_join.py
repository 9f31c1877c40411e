"""B200 hash join parity: reference golden vectors, then seeded instances vs
the oracle. Pair ORDER is checked (probe position, then build insertion), which
is stricter than BASELINE's multiset criterion."""

import numpy as np
import pytest

from golden_io import cases
from oracle import oracle
from paper_2601_19911_b200 import FULL_ROW, KeyVector

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", cases("probe"), ids=lambda c: f"{c['tag']}-{len(c['bkeys'])}x{len(c['pkeys'])}")
def test_probe_matches_reference_golden(b200, case):
    res = b200.probe(KeyVector(case["bkeys"], case["brows"]), KeyVector(case["pkeys"], case["prows"]))
    assert res.payload.probe_rows.tolist() == case["exp_p"].tolist()
    assert res.payload.build_rows.tolist() == case["exp_b"].tolist()
    assert res.payload.probe_count == len(case["pkeys"])
    assert res.ledger.h2d_bytes == 12 * (len(case["bkeys"]) + len(case["pkeys"]))
    assert res.ledger.d2h_bytes == 8 * len(case["exp_p"])


@pytest.mark.parametrize("nb,np_,domain", [
    (1_000_000, 10_000_000, 2_000_000),   # config C2 shape
    (100_000, 1_000_000, 200_000),
    (50_000, 300_000, 5_000),             # groups of ~10
    (200_000, 100_000, 300),              # groups of ~670 (block sort path)
    (60_000, 5_000, 2),                   # groups of ~30000 (global in-place sort path)
    (1, 100_000, 2),
    (100_000, 1, 2),
])
def test_probe_random_vs_oracle(b200, nb, np_, domain):
    rng = np.random.default_rng(nb + np_ + domain)
    bk = rng.integers(0, domain, size=nb).astype(np.float64)
    pk = rng.integers(0, domain, size=np_).astype(np.float64)
    br = rng.permutation(nb).astype(np.uint32)
    pr = rng.permutation(np_).astype(np.uint32)
    res = b200.probe(KeyVector(bk, br), KeyVector(pk, pr))
    ep, eb = oracle.join(bk, br, pk, pr)
    assert np.array_equal(res.payload.probe_rows, ep)
    assert np.array_equal(res.payload.build_rows, eb)


def test_probe_more_pairs_than_probes_grows_output(b200):
    rng = np.random.default_rng(4)
    bk = rng.integers(0, 4, size=20_000).astype(np.float64)  # ~5000 matches per probe
    pk = rng.integers(0, 4, size=3000).astype(np.float64)
    br = np.arange(20_000, dtype=np.uint32)
    pr = np.arange(3000, dtype=np.uint32)
    res = b200.probe(KeyVector(bk, br), KeyVector(pk, pr))
    ep, eb = oracle.join(bk, br, pk, pr)
    assert res.payload.match_count == len(ep) > 3000
    assert np.array_equal(res.payload.probe_rows, ep) and np.array_equal(res.payload.build_rows, eb)


def test_probe_signed_zero_negative_and_extreme_keys(b200):
    bk = np.array([0.0, -0.0, -1e300, 1e300, 5e-324, -5e-324, -7.25, 0.0])
    pk = np.array([-0.0, 1e300, -7.25, 5e-324, 3.0, 0.0])
    br = np.arange(len(bk), dtype=np.uint32) * 3
    pr = np.arange(len(pk), dtype=np.uint32) + 100
    res = b200.probe(KeyVector(bk, br), KeyVector(pk, pr))
    ep, eb = oracle.join(bk, br, pk, pr)
    assert res.payload.matches == list(zip(ep.tolist(), eb.tolist()))


def test_probe_full_row_mode(b200):
    rng = np.random.default_rng(3)
    b = KeyVector(rng.integers(0, 100, size=5000).astype(np.float64), np.arange(5000))
    p = KeyVector(rng.integers(0, 100, size=20_000).astype(np.float64), np.arange(20_000))
    full = b200.probe(b, p, mode=FULL_ROW, payload_bytes=188)
    key = b200.probe(b, p)
    assert full.payload.matches == key.payload.matches
    assert full.ledger.h2d_bytes == 196 * 25_000


def test_join_resident_api(cuda):
    import torch

    from paper_2601_19911_b200 import resident

    rng = np.random.default_rng(11)
    nb, np_ = 300_000, 2_000_000
    bk = rng.integers(0, 600_000, size=nb).astype(np.float64)
    pk = rng.integers(0, 600_000, size=np_).astype(np.float64)
    br = rng.permutation(nb).astype(np.uint32)
    pr = rng.permutation(np_).astype(np.uint32)
    t = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).to(cuda)  # noqa: E731
    op, ob = resident.join(t(bk), t(br), t(pk), t(pr))
    ep, eb = oracle.join(bk, br, pk, pr)
    assert np.array_equal(op.cpu().numpy().view(np.uint32), ep)
    assert np.array_equal(ob.cpu().numpy().view(np.uint32), eb)
    # capacity contract: too-small buffers -> CapacityError with the true count
    from paper_2601_19911_b200 import CapacityError

    resident.join_build(t(bk), t(br))
    small = torch.empty(10, dtype=torch.int32, device=cuda)
    with pytest.raises(CapacityError):
        resident.join_probe(t(pk), t(pr), small, small.clone())


@pytest.mark.parametrize("dense", [True, False])
def test_join_graph_replay_and_profiling_levels(cuda, dense):
    """The resident build + async probe captured in CUDA graphs (as bench.py
    replays them) gives the oracle's pairs on every replay, with the density flag
    alternating between builds; profiling level 2 times the probe, not the build."""
    import torch

    from paper_2601_19911_b200 import _native, resident

    rng = np.random.default_rng(31 + dense)
    nb, np_ = 400_000, 2_000_000
    bk = rng.integers(0, 800_000, size=nb).astype(np.float64)
    pk = rng.integers(0, 800_000, size=np_).astype(np.float64)
    br = np.arange(nb, dtype=np.uint32) + 7 if dense else rng.permutation(nb).astype(np.uint32)
    pr = np.arange(np_, dtype=np.uint32)
    t = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).to(cuda)  # noqa: E731
    tbk, tbr, tpk, tpr = t(bk), t(br), t(pk), t(pr)
    ep, eb = oracle.join(bk, br, pk, pr)
    out_p = torch.empty(len(ep) + 16, dtype=torch.int32, device=cuda)
    out_b = torch.empty_like(out_p)
    m = torch.zeros(1, dtype=torch.int64, device=cuda)
    resident.set_profiling(True, build_start=False)
    try:
        resident.join_build(tbk, tbr)
        resident.join_probe_async(tpk, tpr, out_p, out_b, m)
        torch.cuda.synchronize()
        kt = _native.kernel_times()
        assert kt["join_build_ms"] == 0.0 and kt["join_probe_ms"] > 0.0
    finally:
        resident.set_profiling(False)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        gb, gp = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gb):
            resident.join_build(tbk, tbr)
        with torch.cuda.graph(gp):
            resident.join_probe_async(tpk, tpr, out_p, out_b, m)
    for _ in range(3):
        out_p.fill_(-1)
        gb.replay()
        gp.replay()
        torch.cuda.synchronize()
        assert int(m.item()) == len(ep)
        assert np.array_equal(out_p[: len(ep)].cpu().numpy().view(np.uint32), ep)
        assert np.array_equal(out_b[: len(ep)].cpu().numpy().view(np.uint32), eb)


# ---- radix-partitioned join (tables larger than two slices) -------------------
# GOLP_JOIN_SLICE_BYTES shrinks the slice so small builds take the partitioned
# path; GOLP_JOIN_PART_PROBE=1 forces the slice-ordered probe as well.
@pytest.mark.parametrize("slice_bytes", [64, 1024, 65536])
@pytest.mark.parametrize("part_probe", ["0", "1"])
@pytest.mark.parametrize("nb,np_,domain", [
    (100_000, 1_000_000, 200_000),
    (50_000, 300_000, 5_000),
    (200_000, 100_000, 300),
    (5000, 70_000, 1 << 40),
])
def test_partitioned_join_vs_oracle(b200, monkeypatch, slice_bytes, part_probe, nb, np_, domain):
    from paper_2601_19911_b200 import _native

    monkeypatch.setenv("GOLP_JOIN_SLICE_BYTES", str(slice_bytes))
    monkeypatch.setenv("GOLP_JOIN_PART_PROBE", part_probe)
    rng = np.random.default_rng(nb ^ np_ ^ slice_bytes)
    bk = rng.integers(0, domain, size=nb).astype(np.float64)
    pk = np.concatenate([rng.choice(bk, size=np_ // 2), rng.integers(0, domain, size=np_ - np_ // 2)])
    rng.shuffle(pk)
    br = rng.permutation(nb).astype(np.uint32)
    pr = rng.permutation(np_).astype(np.uint32)
    _native.check(_native.load().golp_set_profiling(1))
    try:
        res = b200.probe(KeyVector(bk, br), KeyVector(pk, pr))
        kt = _native.kernel_times()
    finally:
        _native.check(_native.load().golp_set_profiling(0))
    assert kt["join_slices"] > 1
    ep, eb = oracle.join(bk, br, pk, pr)
    assert np.array_equal(res.payload.probe_rows, ep)
    assert np.array_equal(res.payload.build_rows, eb)


def test_partitioned_join_resident_subchunks(cuda, monkeypatch):
    import torch

    from paper_2601_19911_b200 import resident

    monkeypatch.setenv("GOLP_JOIN_SLICE_BYTES", "65536")
    monkeypatch.setenv("GOLP_JOIN_PART_PROBE", "1")
    rng = np.random.default_rng(5)
    nb, np_ = 400_000, 3_000_000
    bk = rng.integers(0, 800_000, size=nb).astype(np.float64)
    pk = rng.integers(0, 800_000, size=np_).astype(np.float64)
    br = rng.permutation(nb).astype(np.uint32)
    pr = rng.permutation(np_).astype(np.uint32)
    t = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).to(cuda)  # noqa: E731
    op, ob = resident.join(t(bk), t(br), t(pk), t(pr))
    ep, eb = oracle.join(bk, br, pk, pr)
    assert np.array_equal(op.cpu().numpy().view(np.uint32), ep)
    assert np.array_equal(ob.cpu().numpy().view(np.uint32), eb)


@pytest.mark.parametrize("layout", ["slice", "exact"])
@pytest.mark.parametrize("span", ["4096", "12288"])
def test_partitioned_join_multi_span(b200, monkeypatch, span, layout):
    """Probe sides longer than a span are partitioned span by span; pair offsets
    chain across spans and sub-chunks (each partition layout)."""
    monkeypatch.setenv("GOLP_JOIN_SLICE_BYTES", "4096")
    monkeypatch.setenv("GOLP_JOIN_PART_PROBE", "1")
    monkeypatch.setenv("GOLP_JOIN_SPAN", span)
    if layout == "exact":
        monkeypatch.setenv("GOLP_PART_CAP", "0")
    rng = np.random.default_rng(int(span))
    nb, np_ = 40_000, 90_001
    bk = rng.integers(0, 60_000, size=nb).astype(np.float64)
    pk = rng.integers(0, 60_000, size=np_).astype(np.float64)
    br = rng.permutation(nb).astype(np.uint32)
    pr = rng.permutation(np_).astype(np.uint32)
    res = b200.probe(KeyVector(bk, br), KeyVector(pk, pr))
    ep, eb = oracle.join(bk, br, pk, pr)
    assert np.array_equal(res.payload.probe_rows, ep)
    assert np.array_equal(res.payload.build_rows, eb)


@pytest.mark.parametrize("hot", [0.0, 0.3, 0.97, 1.0])
def test_partitioned_probe_hot_key_overflows_slice(b200, monkeypatch, hot):
    """Probe sides whose slices are far from balanced (one key is 30% .. 100%
    of the probes): the fixed-capacity slice of the hot key overflows and its
    runs go to the overflow area; pairs and order must not change."""
    monkeypatch.setenv("GOLP_JOIN_SLICE_BYTES", "65536")
    monkeypatch.setenv("GOLP_JOIN_PART_PROBE", "1")
    rng = np.random.default_rng(int(hot * 100))
    nb, np_ = 60_000, 400_000
    bk = rng.integers(0, 120_000, size=nb).astype(np.float64)
    nhot = int(np_ * hot)
    pk = np.concatenate([np.full(nhot, bk[7]), rng.integers(0, 120_000, size=np_ - nhot).astype(np.float64)])
    pk = rng.permutation(pk)
    br = rng.permutation(nb).astype(np.uint32)
    pr = np.arange(np_, dtype=np.uint32)
    res = b200.probe(KeyVector(bk, br), KeyVector(pk, pr))
    ep, eb = oracle.join(bk, br, pk, pr)
    assert res.payload.match_count == len(ep)
    assert np.array_equal(res.payload.probe_rows, ep) and np.array_equal(res.payload.build_rows, eb)


@pytest.mark.parametrize("rows_kind", ["high", "mixed", "dense_high_base"])
def test_two_member_groups_with_large_row_ids(b200, rows_kind):
    """Key groups of two keep both rows in the slot only when the second row
    fits 30 bits; row ids at and above 2^30 take the side-array path, and a
    dense column starting near 2^32 keeps positions. Pairs and order must match."""
    rng = np.random.default_rng(len(rows_kind))
    nb, np_ = 300_000, 1_000_000
    bk = rng.integers(0, 400_000, size=nb).astype(np.float64)  # many groups of two
    if rows_kind == "high":
        br = rng.choice(np.arange(1 << 30, (1 << 32) - 1, dtype=np.uint64), size=nb, replace=False).astype(np.uint32)
    elif rows_kind == "mixed":
        br = rng.permutation(nb).astype(np.uint32)
        br[rng.random(nb) < 0.5] |= np.uint32(1 << 30)
    else:
        br = (np.arange(nb, dtype=np.uint64) + ((1 << 32) - nb - 5)).astype(np.uint32)
    pk = rng.integers(0, 400_000, size=np_).astype(np.float64)
    pr = np.arange(np_, dtype=np.uint32)
    res = b200.probe(KeyVector(bk, br), KeyVector(pk, pr))
    ep, eb = oracle.join(bk, br, pk, pr)
    assert res.payload.match_count == len(ep)
    assert np.array_equal(res.payload.probe_rows, ep) and np.array_equal(res.payload.build_rows, eb)


def test_partitioned_join_natural_scale(cuda):
    """A table above the partitioning threshold with default settings (1 GiB
    table, 64 slices, probe side partitioned) against the oracle."""
    import torch

    from paper_2601_19911_b200 import _native, resident

    rng = np.random.default_rng(21)
    nb, np_ = 20_000_000, 60_000_000
    bk = rng.integers(0, 2 * nb, size=nb).astype(np.float64)
    pk = rng.integers(0, 2 * nb, size=np_).astype(np.float64)
    br = rng.permutation(nb).astype(np.uint32)
    pr = np.arange(np_, dtype=np.uint32)
    t = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).to(cuda)  # noqa: E731
    resident.set_profiling(True)
    try:
        op, ob = resident.join(t(bk), t(br), t(pk), t(pr))
        kt = _native.kernel_times()
    finally:
        resident.set_profiling(False)
    assert kt["join_slices"] > 1
    ep, eb = oracle.join(bk, br, pk, pr)
    assert np.array_equal(op.cpu().numpy().view(np.uint32), ep)
    assert np.array_equal(ob.cpu().numpy().view(np.uint32), eb)


def _mix64(z):
    z = z.astype(np.uint64)
    z ^= z >> np.uint64(30)
    z *= np.uint64(0xBF58476D1CE4E5B9)
    z ^= z >> np.uint64(27)
    z *= np.uint64(0x94D049BB133111EB)
    z ^= z >> np.uint64(31)
    return z


@pytest.mark.parametrize("where", ["slice_end", "table_end", "one_slice_overfull"])
def test_probe_keys_crowding_a_slice_boundary(b200, where):
    """Build keys chosen (through mix64) to crowd a few home slots -- at the end
    of a 2048-slot region, at the end of the table (walks wrap to slot 0), or
    2600 keys homed in one quarter of the table: long linear-probing walks, and
    groups of up to ~60 members exercise every group path."""
    nb_rand = 3000
    cap = 8192  # pow2 >= 2 * nb for nb in (2048, 4096]
    cand = np.arange(1, 3_000_000, dtype=np.float64)
    home = (_mix64(cand.view(np.uint64)) & np.uint64(cap - 1)) & ~np.uint64(1)
    if where == "slice_end":
        pick = cand[(home >= 2048 - 8) & (home < 2048)][:120]
    elif where == "table_end":
        pick = cand[home >= cap - 8][:120]
    else:  # far more keys than a 2048-slot slice holds
        pick = cand[home < 2048][:2600]
    rng = np.random.default_rng(len(pick))
    reps = rng.integers(1, 60, size=len(pick)) if where != "one_slice_overfull" else np.ones(len(pick), np.int64)
    crowd = np.repeat(pick, reps)
    nb = min(len(crowd), 4000)
    filler = rng.integers(5_000_000, 6_000_000, size=max(0, 4000 - nb)).astype(np.float64)
    bk = rng.permutation(np.concatenate([crowd[:nb], filler]))
    assert 2048 < len(bk) <= 4096
    br = rng.permutation(len(bk)).astype(np.uint32)
    pk = np.concatenate([pick, filler[:500], rng.integers(0, 7_000_000, size=3000).astype(np.float64)])
    pk = rng.permutation(pk)
    pr = np.arange(len(pk), dtype=np.uint32)
    res = b200.probe(KeyVector(bk, br), KeyVector(pk, pr))
    ep, eb = oracle.join(bk, br, pk, pr)
    assert res.payload.match_count == len(ep)
    assert np.array_equal(res.payload.probe_rows, ep) and np.array_equal(res.payload.build_rows, eb)


@pytest.mark.parametrize("rows_kind", ["dense_offset", "one_swap", "permuted"])
def test_join_build_row_column_density_check(cuda, rows_kind):
    """Build sides of >= 4 Mi entries go through the on-device dense-row check:
    a dense column lets the build skip the position -> row gathers, anything else
    must keep them. Groups of every size class appear (domain = nb / 2)."""
    import torch

    from paper_2601_19911_b200 import resident

    rng = np.random.default_rng(23)
    nb, np_ = 5_000_000, 1_000_000
    bk = rng.integers(0, nb // 2, size=nb).astype(np.float64)
    pk = rng.integers(0, nb // 2, size=np_).astype(np.float64)
    br = np.arange(nb, dtype=np.uint32) + 77
    if rows_kind == "one_swap":
        br[[nb - 3, nb - 2]] = br[[nb - 2, nb - 3]]
    elif rows_kind == "permuted":
        br = rng.permutation(br)
    pr = np.arange(np_, dtype=np.uint32)
    t = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).to(cuda)  # noqa: E731
    op, ob = resident.join(t(bk), t(br), t(pk), t(pr))
    ep, eb = oracle.join(bk, br, pk, pr)
    assert np.array_equal(op.cpu().numpy().view(np.uint32), ep)
    assert np.array_equal(ob.cpu().numpy().view(np.uint32), eb)


@pytest.mark.parametrize("offset", [1, 2])
def test_partitioned_join_misaligned_key_columns(cuda, monkeypatch, offset):
    """Key columns that start 8 bytes off a 16-byte boundary (tensor views) take
    the partition scatter's plain-load path instead of the TMA bulk copies; both
    sides, every tile, same answer."""
    import torch

    from paper_2601_19911_b200 import resident

    monkeypatch.setenv("GOLP_JOIN_SLICE_BYTES", "65536")
    monkeypatch.setenv("GOLP_JOIN_PART_PROBE", "1")
    rng = np.random.default_rng(31 + offset)
    nb, np_ = 300_000, 1_000_000
    bk = rng.integers(0, 600_000, size=nb + offset).astype(np.float64)
    pk = rng.integers(0, 600_000, size=np_ + offset).astype(np.float64)
    br = rng.permutation(nb).astype(np.uint32)
    pr = rng.permutation(np_).astype(np.uint32)
    t = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).to(cuda)  # noqa: E731
    tbk, tpk = t(bk)[offset:], t(pk)[offset:]
    assert (tbk.data_ptr() % 16 != 0) == (offset % 2 == 1)
    op, ob = resident.join(tbk, t(br), tpk, t(pr))
    ep, eb = oracle.join(bk[offset:], br, pk[offset:], pr)
    assert np.array_equal(op.cpu().numpy().view(np.uint32), ep)
    assert np.array_equal(ob.cpu().numpy().view(np.uint32), eb)


def test_resident_topk_and_sort_misaligned_views(cuda):
    """Top-K and the full sort over key / row views that start off a 16-byte
    boundary (vector loads must not assume the allocation's alignment)."""
    import torch

    from paper_2601_19911_b200 import resident

    rng = np.random.default_rng(37)
    n = 3_000_001
    keys = rng.integers(0, 1 << 40, size=n + 1).astype(np.float64)
    rows = rng.permutation(n + 1).astype(np.uint32)
    tk = torch.from_numpy(keys).to(cuda)[1:]
    tr = torch.from_numpy(rows.view(np.int32)).to(cuda)[1:]
    got = resident.topk(tk, tr, 777)
    got = (got[0] if isinstance(got, tuple) else got).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, oracle.topk(keys[1:], rows[1:], 777))
    srt = resident.full_sort(tk, tr).cpu().numpy().view(np.uint32)
    assert np.array_equal(srt, rows[1:][np.lexsort((rows[1:], keys[1:]))])


@pytest.mark.parametrize("part_probe,span", [("0", None), ("1", None), ("1", "12288")])
@pytest.mark.parametrize("base", [0, 1000, (1 << 32) - 2_000_000])
def test_join_probe_positions_vs_oracle(cuda, monkeypatch, part_probe, span, base):
    """Probe row ids given as positions (golp_join_probe_device_positions[_async]):
    the same pairs, in the same order, as the explicit row column."""
    import torch

    from paper_2601_19911_b200 import resident

    monkeypatch.setenv("GOLP_JOIN_PART_PROBE", part_probe)
    if part_probe == "1":
        monkeypatch.setenv("GOLP_JOIN_SLICE_BYTES", "65536")
    if span:
        monkeypatch.setenv("GOLP_JOIN_SPAN", span)
    rng = np.random.default_rng(base % 1000 + 3)
    nb, np_ = 300_000, 2_000_000
    bk = rng.integers(0, 600_000, size=nb).astype(np.float64)
    pk = rng.integers(0, 600_000, size=np_).astype(np.float64)
    br = rng.permutation(nb).astype(np.uint32)
    pr = (np.arange(np_, dtype=np.uint64) + base).astype(np.uint32)
    t = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).to(cuda)  # noqa: E731
    ep, eb = oracle.join(bk, br, pk, pr)
    op, ob = resident.join(t(bk), t(br), t(pk), base)
    assert np.array_equal(op.cpu().numpy().view(np.uint32), ep)
    assert np.array_equal(ob.cpu().numpy().view(np.uint32), eb)
    out_p = torch.empty(len(ep) + 16, dtype=torch.int32, device=cuda)
    out_b = torch.empty_like(out_p)
    m = torch.zeros(1, dtype=torch.int64, device=cuda)
    resident.join_build(t(bk), t(br))
    resident.join_probe_async(t(pk), base, out_p, out_b, m)
    torch.cuda.synchronize()
    assert int(m.item()) == len(ep)
    assert np.array_equal(out_p[: len(ep)].cpu().numpy().view(np.uint32), ep)
    assert np.array_equal(out_b[: len(ep)].cpu().numpy().view(np.uint32), eb)


def test_join_probe_positions_bounds(cuda):
    import torch

    from paper_2601_19911_b200 import _native, resident

    pk = torch.zeros(1000, dtype=torch.float64, device=cuda)
    resident.join_build(pk[:10].clone(), torch.arange(10, dtype=torch.int32, device=cuda))
    out = torch.empty(10, dtype=torch.int32, device=cuda)
    with pytest.raises(ValueError):
        resident.join_probe(pk, (1 << 32) - 999, out, out.clone())
    lib = _native.load()
    m = torch.zeros(1, dtype=torch.int64, device=cuda)
    assert lib.golp_join_probe_device_positions_async(pk.data_ptr(), 1000, (1 << 32) - 999, out.data_ptr(),
                                                      out.data_ptr(), 10, m.data_ptr(), 0) != 0
    assert lib.golp_join_probe_device_async(pk.data_ptr(), 0, 1000, out.data_ptr(), out.data_ptr(), 10,
                                            m.data_ptr(), 0) != 0  # null row column
