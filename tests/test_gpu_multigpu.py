"""Multi-GPU paths on the hardware this run has.

* B200Device(devices=[...]) shards every host-buffer call over several
  contexts, one host thread each: Top-K over contiguous key ranges + merge of the
  local top-K lists, join with the build side on every context and the probe
  side split. With one visible GPU the shards are independent contexts on that
  GPU (devices=[0, 0, 0]); the sharding, merge and pair concatenation are the
  same code a G-GPU box runs. Results must be the reference's, order included.
* With >= 2 visible GPUs: B200Device(gpus=2) and the NCCL exchange of
  sharded.py under torch.distributed (one process per GPU).
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle
from paper_2601_19911_b200 import B200Device, KeyVector

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sharded_dev(cuda):
    dev = B200Device(devices=[0, 0, 0])
    yield dev
    dev.close()


@pytest.mark.parametrize("n,k,domain", [(1_000_000, 100, 1 << 50), (3_000_000, 1000, 5000), (2, 10, 10),
                                        (100_000, 60_000, 1 << 20), (7_000_000, 100_000, 1 << 30)])
def test_sharded_topk_matches_oracle(sharded_dev, n, k, domain):
    rng = np.random.default_rng(n + k)
    keys = rng.integers(0, domain, n).astype(np.float64)
    rows = rng.permutation(n).astype(np.uint32)
    res = sharded_dev.topk(KeyVector(keys, rows), k)
    np.testing.assert_array_equal(res.payload.rows, oracle.topk(keys, rows, k))
    led = res.ledger
    assert led.h2d_bytes == 12 * n and led.d2h_bytes == 4 * min(k, n)
    assert abs(led.total - (led.t_h2d + led.t_kernel + led.t_d2h + led.t_post)) < 1e-12


@pytest.mark.parametrize("nb,np_,domain", [(10_000, 100_000, 20_000), (1_000_000, 10_000_000, 2_000_000),
                                           (50, 5, 10), (3_000, 200_000, 300)])
def test_sharded_probe_matches_oracle_in_reference_order(sharded_dev, nb, np_, domain):
    rng = np.random.default_rng(nb + np_)
    bk = rng.integers(0, domain, nb).astype(np.float64)
    pk = rng.integers(0, domain, np_).astype(np.float64)
    br = rng.permutation(nb).astype(np.uint32)
    pr = rng.permutation(np_).astype(np.uint32)
    res = sharded_dev.probe(KeyVector(bk, br), KeyVector(pk, pr))
    ep, eb = oracle.join(bk, br, pk, pr)
    np.testing.assert_array_equal(res.payload.probe_rows, ep)
    np.testing.assert_array_equal(res.payload.build_rows, eb)
    assert res.ledger.d2h_bytes == 8 * len(ep) and res.ledger.h2d_bytes == 12 * (nb + np_)


def test_sharded_device_through_the_gate_and_a_profile_per_g(sharded_dev):
    """The gate runs unchanged on a sharded device; calibrate_device_profile gives
    the G-shard profile (the reference's model has no G term, device.py:154-181)."""
    from paper_2601_19911_b200 import DEVICE, OP_PROBE, OP_TOPK, GateConfig, execute_path, generate_table
    from paper_2601_19911_b200.harness import calibrate_device_profile

    t = generate_table(2_000_000, 8, seed=4)
    r, lat = execute_path(t, OP_TOPK, 500, GateConfig(), sharded_dev, DEVICE)
    np.testing.assert_array_equal(r.row_ids, oracle.topk(t.key_column, t.positions, 500))
    bt = generate_table(20_000, 8, seed=5)
    p, _ = execute_path((bt, t), OP_PROBE, 1, GateConfig(), sharded_dev, DEVICE)
    assert p.probe_count == t.row_count
    prof = calibrate_device_profile(sharded_dev, ns=(200_000, 1_000_000, 4_000_000), repeats=2)
    assert prof.kernel_rate_topk > 1e-12 and prof.h2d_bandwidth > 1e9


def test_context_isolation_and_device_pointer_check(cuda):
    """A resident call with a tensor on another device is refused, not run on
    this context's device (the round-1 single-context library ran it silently)."""
    import torch

    from paper_2601_19911_b200 import _native

    lib = _native.load()
    assert lib.golp_use_device(0) == _native.GOLP_OK
    if torch.cuda.device_count() < 2:
        assert lib.golp_use_device(torch.cuda.device_count() + 3) != _native.GOLP_OK
        return
    t = torch.zeros(16, dtype=torch.float64, device="cuda:1")
    r = torch.zeros(16, dtype=torch.int32, device="cuda:1")
    out = torch.zeros(4, dtype=torch.int32, device="cuda:1")
    rc = lib.golp_topk_device(t.data_ptr(), r.data_ptr(), 16, 4, out.data_ptr(), 0, 0)
    assert rc == _native.GOLP_ERR_INVALID


def _need_two_gpus():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 visible GPUs (this run's boxes have one)")


def test_two_gpus_in_one_process(cuda):
    _need_two_gpus()
    rng = np.random.default_rng(7)
    keys = rng.standard_normal(5_000_000)
    rows = np.arange(5_000_000, dtype=np.uint32)
    with B200Device(gpus=2) as dev:
        assert dev.gpus == 2
        got = dev.topk(KeyVector(keys, rows), 1000).payload.rows
    np.testing.assert_array_equal(got, oracle.topk(keys, rows, 1000))


def _nccl_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2601_19911_b200 import sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    rng = np.random.default_rng(11)
    n = 4_000_000
    keys = rng.integers(0, 1 << 20, n).astype(np.float64)
    rows = np.arange(n, dtype=np.uint32)
    lo, hi = sharded.shard_bounds(n, world, rank)
    dev = torch.device("cuda", rank)
    out = sharded.topk(torch.from_numpy(keys[lo:hi]).to(dev), torch.from_numpy(rows[lo:hi].view(np.int32)).to(dev),
                       5000)
    bk = rng.integers(0, 100_000, 50_000).astype(np.float64)
    pk = rng.integers(0, 100_000, 1_000_000).astype(np.float64)
    blo, bhi = sharded.shard_bounds(len(bk), world, rank)
    plo, phi = sharded.shard_bounds(len(pk), world, rank)
    pairs = sharded.join(torch.from_numpy(bk[blo:bhi]).to(dev),
                         torch.arange(blo, bhi, dtype=torch.int32, device=dev),
                         torch.from_numpy(pk[plo:phi]).to(dev), torch.arange(plo, phi, dtype=torch.int32, device=dev))
    p, b = sharded.gather_pairs(pairs)
    if rank == 0:
        ep, eb = oracle.join(bk, np.arange(len(bk), dtype=np.uint32), pk, np.arange(len(pk), dtype=np.uint32))
        q.put(bool(np.array_equal(out.cpu().numpy().view(np.uint32), oracle.topk(keys, rows, 5000))
                   and np.array_equal(p.cpu().numpy().view(np.uint32), ep)
                   and np.array_equal(b.cpu().numpy().view(np.uint32), eb)))
    dist.destroy_process_group()


def test_nccl_exchange_two_ranks(cuda):
    _need_two_gpus()
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_nccl_worker, args=(2, 29517, q), nprocs=2, join=True, start_method="spawn")
    assert q.get(timeout=60)
