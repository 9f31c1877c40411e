"""Multi-GPU sharding: one process per GPU, torch.distributed for the exchange.

Top-K: each rank owns a contiguous position range, computes its
local top-K' under the total order (key desc, row asc) on its GPU, the
encoded (key code, row) candidates are all-gathered over NVLink (NCCL), and
every rank merges the G*K' candidates with the same select engine. Correct
because the union of local top-K sets contains the global top-K under a total
order -- the GPU analogue of ProxyDevice's chunk -> merge
(pkg/src/golp/device.py:354-363).

Join: the build side is replicated -- each rank contributes its contiguous
build shard, an all-gather in rank order reassembles the build column in
global position order (so insertion order, and hence pair order, is the
reference's), every rank builds the full table and probes its own contiguous
probe shard. Concatenating the per-rank pair lists in rank order gives exactly
host_hash_probe's order (probe position, then build insertion position).

The per-rank compute is an `engine` object (default: the CUDA engine in
resident.py). Tests substitute a CPU engine to exercise this exchange logic
with the gloo backend.
"""

from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


class CudaEngine:
    """Per-rank kernels of libgolp_b200 (device-resident inputs)."""

    def topk(self, keys, rows, k):
        from . import resident

        return resident.topk(keys, rows, k, want_codes=True)

    def merge(self, codes, rows, k):
        from . import resident

        out, oc = resident.merge(codes, rows, k, want_codes=True)
        return out, oc

    def join(self, bkeys, brows, pkeys, prows):
        from . import resident

        return resident.join(bkeys, brows, pkeys, prows)


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous position range [lo, hi) of `rank` among `world` (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _all_gather_ragged(t: torch.Tensor, group=None) -> list[torch.Tensor]:
    """all_gather of 1-D tensors whose lengths differ per rank (rank order)."""
    world = dist.get_world_size(group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(sizes) if sizes else 0
    padded = torch.zeros(cap, dtype=t.dtype, device=t.device)
    padded[: t.numel()] = t
    bufs = [torch.empty(cap, dtype=t.dtype, device=t.device) for _ in range(world)]
    dist.all_gather(bufs, padded, group=group)
    return [b[:s] for b, s in zip(bufs, sizes)]


def topk(keys: torch.Tensor, rows: torch.Tensor, k: int, group=None, engine=None):
    """Global top-k over all ranks' local (keys, rows) shards.

    Returns the row ids (int32 storage of u32) best first, identical on every rank.
    """
    if k < 1:
        raise ValueError("k must be at least 1")
    eng = engine or CudaEngine()
    local_rows, local_codes = eng.topk(keys, rows, k)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local_rows
    codes = torch.cat(_all_gather_ragged(local_codes, group))
    cand_rows = torch.cat(_all_gather_ragged(local_rows, group))
    if codes.numel() == 0:
        return cand_rows
    out, _ = eng.merge(codes, cand_rows, k)
    return out


def join(build_keys: torch.Tensor, build_rows: torch.Tensor, probe_keys: torch.Tensor, probe_rows: torch.Tensor,
         group=None, engine=None):
    """Replicated-build, sharded-probe join.

    build_* is this rank's contiguous build shard, probe_* its probe shard.
    Returns this rank's (probe_rows, build_rows) pairs; concatenated in rank
    order they are the reference's single-node output.
    """
    eng = engine or CudaEngine()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        build_keys = torch.cat(_all_gather_ragged(build_keys, group))
        build_rows = torch.cat(_all_gather_ragged(build_rows, group))
    return eng.join(build_keys, build_rows, probe_keys, probe_rows)


def gather_pairs(pairs: tuple[torch.Tensor, torch.Tensor], group=None) -> Optional[tuple[torch.Tensor, torch.Tensor]]:
    """Concatenate every rank's pairs in rank order (all ranks receive them)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return pairs
    p = torch.cat(_all_gather_ragged(pairs[0], group))
    b = torch.cat(_all_gather_ragged(pairs[1], group))
    return p, b
