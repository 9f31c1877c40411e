"""World-size-2 gloo runs of the multi-GPU exchange logic (sharded.py) on CPU.

The per-rank kernels are replaced by a CPU engine built on the oracle, so what
is tested here is the sharding, the all-gathers (ragged, rank-ordered) and the
merge/concatenation order -- the parts that are the same on N B200s.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle


def _codes(keys: np.ndarray) -> np.ndarray:
    b = (np.asarray(keys, dtype=np.float64) + 0.0).view(np.uint64)
    sign = (b >> np.uint64(63)).astype(bool)
    return np.where(sign, ~b, b | np.uint64(1 << 63))


class CpuEngine:
    def topk(self, keys, rows, k):
        kn, rn = keys.numpy(), rows.numpy().view(np.uint32)
        out = oracle.topk(kn, rn, k)
        pos = {int(r): i for i, r in enumerate(rn.tolist())}
        codes = _codes(kn[[pos[int(r)] for r in out.tolist()]]) if len(out) else np.empty(0, np.uint64)
        return torch.from_numpy(out.view(np.int32).copy()), torch.from_numpy(codes.view(np.int64).copy())

    def merge(self, codes, rows, k):
        c = codes.numpy().view(np.uint64)
        r = rows.numpy().view(np.uint32)
        order = np.lexsort((r, ~c))  # code desc, row asc
        take = order[:k]
        return torch.from_numpy(r[take].view(np.int32).copy()), torch.from_numpy(c[take].view(np.int64).copy())

    def join(self, bkeys, brows, pkeys, prows):
        p, b = oracle.join(bkeys.numpy(), brows.numpy().view(np.uint32), pkeys.numpy(), prows.numpy().view(np.uint32))
        return torch.from_numpy(p.view(np.int32)), torch.from_numpy(b.view(np.int32))


def _worker(rank, world, port, q):
    from paper_2601_19911_b200 import sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(123)
        n = 50_001
        keys = rng.integers(0, 500, size=n).astype(np.float64)  # heavy ties across the shard edge
        rows = rng.permutation(n).astype(np.uint32)
        lo, hi = sharded.shard_bounds(n, world, rank)
        out = {}
        for k in (1, 100, 30_000):
            got = sharded.topk(torch.from_numpy(keys[lo:hi]), torch.from_numpy(rows[lo:hi].view(np.int32)), k,
                               engine=CpuEngine())
            out[f"topk{k}"] = got.numpy().view(np.uint32).tolist()
        nb, np_ = 7_001, 20_003
        bk = rng.integers(0, 3000, size=nb).astype(np.float64)
        br = rng.permutation(nb).astype(np.uint32)
        pk = rng.integers(0, 3000, size=np_).astype(np.float64)
        pr = rng.permutation(np_).astype(np.uint32)
        blo, bhi = sharded.shard_bounds(nb, world, rank)
        plo, phi = sharded.shard_bounds(np_, world, rank)
        pairs = sharded.join(torch.from_numpy(bk[blo:bhi]), torch.from_numpy(br[blo:bhi].view(np.int32)),
                             torch.from_numpy(pk[plo:phi]), torch.from_numpy(pr[plo:phi].view(np.int32)),
                             engine=CpuEngine())
        p, b = sharded.gather_pairs(pairs)
        out["join_p"] = p.numpy().view(np.uint32).tolist()
        out["join_b"] = b.numpy().view(np.uint32).tolist()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_topk_and_join_equal_single_node_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get() for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(123)
    n = 50_001
    keys = rng.integers(0, 500, size=n).astype(np.float64)
    rows = rng.permutation(n).astype(np.uint32)
    for k in (1, 100, 30_000):
        expect = oracle.topk(keys, rows, k).tolist()
        for r in range(world):
            assert results[r][f"topk{k}"] == expect
    nb, np_ = 7_001, 20_003
    bk = rng.integers(0, 3000, size=nb).astype(np.float64)
    br = rng.permutation(nb).astype(np.uint32)
    pk = rng.integers(0, 3000, size=np_).astype(np.float64)
    pr = rng.permutation(np_).astype(np.uint32)
    ep, eb = oracle.join(bk, br, pk, pr)
    for r in range(world):
        assert results[r]["join_p"] == ep.tolist()
        assert results[r]["join_b"] == eb.tolist()


def test_shard_bounds_cover_exactly():
    from paper_2601_19911_b200.sharded import shard_bounds

    for n in (0, 1, 7, 100, 12345):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
