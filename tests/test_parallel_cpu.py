"""Multi-process host logic of the partitioned path on CPU (gloo, world 2/4).

Mirrors the reference's determinism tests (test_parallel.py:21-75: band grid
independent of thread count, bit-identical output for any thread count),
restated for ranks: the halo exchange reproduces the whole-frame block, and
strip labels + the all-gathered seam merge reproduce whole-frame labels
exactly.  Per-strip labels come from the oracle (the GPU labeller is covered
by the -m gpu tests); the collective, the plan and the merge are the product
code.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_15121_b200.parallel import StripPlan, exchange_halo, seam_map, shard_range


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _halo_worker(rank, world, port, H, W, halo, q):
    _init(rank, world, port)
    try:
        full = torch.arange(H * W, dtype=torch.float32).reshape(H, W)
        plan = StripPlan(H, W, world, halo)
        r0, r1 = plan.owned(rank)
        block = exchange_halo(full[r0:r1].clone(), plan, rank)
        b0, b1 = plan.block(rank)
        q.put((rank, bool(torch.equal(block, full[b0:b1]))))
    finally:
        dist.destroy_process_group()


def _seam_worker(rank, world, port, p, q):
    from oracle.stereonorm_oracle import label_components
    _init(rank, world, port)
    try:
        H, W = p.shape
        plan = StripPlan(H, W, world, 1)
        r0, r1 = plan.owned(rank)
        local = label_components(p[r0:r1], index_offset=r0 * W)
        keys, vals = seam_map(torch.from_numpy(local.astype(np.int32)), world)
        lut = dict(zip(keys.tolist(), vals.tolist()))
        merged = np.vectorize(lambda v: lut.get(v, v), otypes=[np.int64])(local)
        q.put((rank, merged, keys, vals))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=fn, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


def test_shard_range_partitions():
    for n in (0, 1, 7, 256, 257):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_strip_plan_blocks():
    plan = StripPlan.for_kernel(4320, 7680, 8, 9)
    assert plan.halo == 4
    assert plan.owned(0) == (0, 540) and plan.owned(7) == (3780, 4320)
    assert plan.block(0) == (0, 544) and plan.block(3) == (1616, 2164)
    assert plan.owned_in_block(3) == (4, 544)
    with pytest.raises(ValueError):
        StripPlan(10, 8, 4, 4)  # strips thinner than the halo


@pytest.mark.parametrize("world,H,halo", [(2, 37, 4), (4, 64, 1), (4, 50, 7)])
def test_exchange_halo_gloo(world, H, halo):
    res = _spawn(_halo_worker, world, H, 23, halo)
    assert all(ok for _, ok in res)


@pytest.mark.parametrize("world", [2, 4])
def test_seam_merge_gloo_matches_whole_frame(world):
    from oracle.stereonorm_oracle import label_components
    rng = np.random.default_rng(11 + world)
    H, W = 120, 90
    p = rng.random((H, W)) < 0.57  # near the 8-connected percolation threshold: long seams
    full = label_components(p)
    res = _spawn(_seam_worker, world, p)
    merged = np.concatenate([r[1] for r in res])
    assert np.array_equal(merged, full)
    # the merge map is identical on every rank
    for r in res[1:]:
        assert np.array_equal(r[2], res[0][2]) and np.array_equal(r[3], res[0][3])
