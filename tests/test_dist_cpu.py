"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 path: batch sharding of
the conv workload and row sharding + all-gather of the GEMM result, with the CPU
oracle standing in for the kernels (no GPU here).  Exercises
paper_1810_11066_b200.dist exactly as bench.py uses it."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1810_11066_b200 import dist as bsdist
from paper_1810_11066_b200 import inputs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("total", [1, 7, 8, 256, 1000])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_range_partitions(total, world):
    seen = []
    for r in range(world):
        lo, hi = bsdist.shard_range(total, r, world)
        assert 0 <= lo <= hi <= total
        seen.extend(range(lo, hi))
    assert seen == list(range(total))
    sizes = [bsdist.shard_range(total, r, world)[1] - bsdist.shard_range(total, r, world)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, q):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    try:
        bsdist.init("gloo")
        # row-sharded GEMM + all-gather (BASELINE configs[4] structure)
        m, n, k = 64, 24, 100
        a, w = inputs.dense_operands(m, n, k, 2, 1, seed=5)
        lo, hi = bsdist.shard_range(m, rank, world)
        shard = torch.from_numpy(oracle.dense(a[lo:hi].numpy(), 2, w.numpy(), 1, True))
        full = torch.empty((m, n), dtype=torch.int32)
        bsdist.gather_rows(full, shard)
        ok_gemm = np.array_equal(full.numpy(), oracle.dense(a.numpy(), 2, w.numpy(), 1, True))
        # batch-sharded conv (BASELINE configs[3] structure): no collective; compare own shard
        L = inputs.TABLE1[12]
        act, wt = inputs.conv_operands(L, 4, 2, 1, seed=6)
        blo, bhi = bsdist.shard_range(4, rank, world)
        mine = oracle.conv2d_nhwc(act[blo:bhi].numpy(), 2, wt.numpy(), 1, True, stride=(1, 1), pad=(1, 1))
        ref = oracle.conv2d_nhwc(act.numpy(), 2, wt.numpy(), 1, True, stride=(1, 1), pad=(1, 1))[blo:bhi]
        ok_conv = np.array_equal(mine, ref)
        t = bsdist.max_over_ranks(float(rank + 1))
        bsdist.barrier()
        q.put((rank, ok_gemm, ok_conv, t))
    finally:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


def test_world2_gloo_shard_and_gather():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_gemm, ok_conv, t in res:
        assert ok_gemm and ok_conv
        assert t == float(world)  # max over ranks


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_peer_ranks(world):
    for r in range(world):
        p = bsdist.peer_ranks(r, world)
        assert sorted(p + [r]) == list(range(world)) and len(set(p)) == world - 1


def _fused_worker(rank, world, port, copies, q):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    try:
        bsdist.init("gloo")
        m, n, k = copies.shape[1], copies.shape[2], 96
        a, w = inputs.dense_operands(m, n, k, 2, 1, seed=11)
        lo, hi = bsdist.shard_range(m, rank, world)
        block = torch.from_numpy(oracle.dense(a[lo:hi].numpy(), 2, w.numpy(), 1, True))
        # the fused epilogue's writes: own copy, then every peer's copy, at rows [lo, hi)
        for p in [rank] + bsdist.peer_ranks(rank, world):
            copies[p, lo:hi] = block
        bsdist.barrier()  # the exchange is complete once every rank passed the barrier
        ok = np.array_equal(copies[rank].numpy(), oracle.dense(a.numpy(), 2, w.numpy(), 1, True))
        q.put((rank, ok))
    finally:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_gather_protocol_gloo(world):
    """The protocol of the fused all-gather epilogue (bs_bitserial_dense_tc_prepared_gather
    + dist.FusedGather): each rank stores its row block into every rank's copy of C, then a
    barrier; afterwards every copy is the full product.  Shared CPU tensors stand in for
    the symmetric-memory buffers, the oracle for the kernel."""
    port = _free_port()
    copies = torch.full((world, 50, 12), -1, dtype=torch.int32).share_memory_()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, copies, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)
