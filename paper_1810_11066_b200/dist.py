"""Multi-GPU plumbing of the hot path: one process per GPU,
torch.distributed for process groups and collectives.

* Batch-sharded conv (BASELINE configs[3]): independent images, contiguous blocks per
  rank, weights replicated, no collective on the data path.
* Row-sharded GEMM (BASELINE configs[4]): A rows split across ranks, W replicated,
  one exchange step — an all-gather of the int32 result rows (NCCL over NVLink on
  the GPU box; `gloo` for the CPU tests).

Nothing here computes the method; it only partitions work and moves results.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env():
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 without it)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str, local_rank: int = 0):
    """Initialise the default process group when WORLD_SIZE > 1 (MASTER_ADDR defaults
    to 127.0.0.1)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1 or dist.is_initialized():
        return
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend == "nccl":
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        dist.init_process_group(backend)


def shard_range(total: int, rank: int, world: int):
    """Contiguous block [lo, hi) of `total` units owned by `rank`; blocks differ in size
    by at most one and cover [0, total) exactly once."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def barrier():
    if dist.is_initialized():
        dist.barrier()


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (timing: the job is as slow as its slowest rank)."""
    if not dist.is_initialized():
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(out_full: torch.Tensor, shard: torch.Tensor):
    """All-gather equal-size row shards into out_full ([world * rows][...]); the one
    exchange step of the row-sharded GEMM.  NCCL: all_gather_into_tensor (one
    collective over NVLink/NVSwitch); gloo: all_gather into views of out_full."""
    if not dist.is_initialized():
        out_full.copy_(shard)
        return out_full
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out_full, shard)
    else:
        world = dist.get_world_size()
        parts = list(out_full.chunk(world, dim=0))
        dist.all_gather(parts, shard)
    return out_full


class FusedGather:
    """Buffers of the fused all-gather epilogue: the gathered C [m][n] in
    torch symmetric memory on every rank; this rank's kernel stores its row block
    [lo, hi) into its own copy (local_block) and, over NVLink, into every peer's copy
    (peer_blocks: peer memory mapped into this process); barrier() orders the exchange
    (a device-side barrier on the current stream).  With one process there are no peers
    and C is an ordinary tensor."""

    def __init__(self, m: int, n: int, lo: int, hi: int, device):
        self.lo, self.hi, self.peers, self.handle, self.mc = lo, hi, [], None, 0
        world = dist.get_world_size() if dist.is_initialized() else 1
        if world == 1:
            self.full = torch.empty((m, n), dtype=torch.int32, device=device)
            return
        import torch.distributed._symmetric_memory as symm_mem
        self.full = symm_mem.empty((m, n), dtype=torch.int32, device=device)
        self.handle = symm_mem.rendezvous(self.full, dist.group.WORLD.group_name)
        rank = dist.get_rank()
        self.peers = [self.handle.get_buffer(p, (m, n), torch.int32)[lo:hi] for p in peer_ranks(rank, world)]
        # NVLS multicast (capability probe): torch symmetric memory exposes a multicast address
        # when the GPUs sit on an NVSwitch with multicast support; then the epilogue stores each
        # row segment once with multimem.st (bs_bitserial_dense_tc_prepared_multicast)
        mc = int(getattr(self.handle, "multicast_ptr", 0) or 0)
        self.mc = mc + lo * n * 4 if mc else 0

    def local_block(self):
        return self.full[self.lo:self.hi]

    def peer_blocks(self):
        return self.peers

    def barrier(self):
        if self.handle is not None:
            self.handle.barrier(channel=0)

    def multicast_block(self):
        """Multicast (NVLS) address of this rank's row block, or 0 when unsupported."""
        return self.mc

    def describe(self):
        if self.handle is None:
            return "one process: no peers"
        if self.mc:
            return "torch symmetric memory, NVLS multicast: each row segment stored once with multimem.st"
        return f"torch symmetric memory, {len(self.peers)} peer copies written by the kernel (no multicast support)"


class SingleDeviceMulticast:
    """A multicast (NVLS) object bound to ONE device (CUDA driver API through cuda-python):
    memory reachable through a unicast address and a multicast address, so the multimem
    epilogue can be exercised on a one-GPU box.  Raises RuntimeError when the device or
    driver does not support multicast.  Plumbing only (device memory), no arithmetic."""

    def __init__(self, nbytes: int, device: int = 0):
        from cuda.bindings import driver as drv
        self.drv = drv
        torch.cuda.init()

        def ok(res, what=""):
            err = res[0] if isinstance(res, tuple) else res
            if err != drv.CUresult.CUDA_SUCCESS:
                raise RuntimeError(f"multicast setup failed at {what}: {err}")
            return res[1] if isinstance(res, tuple) and len(res) > 1 else None
        ok(drv.cuInit(0), "cuInit")
        dev = ok(drv.cuDeviceGet(device), "cuDeviceGet")
        if not ok(drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev), "cuDeviceGetAttribute"):
            raise RuntimeError("device reports no multicast support")
        mprop = drv.CUmulticastObjectProp()
        mprop.numDevices = 1
        mprop.handleTypes = drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        mprop.size = nbytes
        gran = ok(drv.cuMulticastGetGranularity(mprop, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity")
        size = (nbytes + gran - 1) // gran * gran
        mprop.size = size
        self.size = size
        self.mc_handle = ok(drv.cuMulticastCreate(mprop), "cuMulticastCreate")
        ok(drv.cuMulticastAddDevice(self.mc_handle, dev), "cuMulticastAddDevice")
        aprop = drv.CUmemAllocationProp()
        aprop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        aprop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        aprop.location.id = device
        aprop.requestedHandleTypes = drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        self.mem = ok(drv.cuMemCreate(size, aprop, 0), "cuMemCreate")
        ok(drv.cuMulticastBindMem(self.mc_handle, 0, self.mem, 0, size, 0), "cuMulticastBindMem")
        acc = drv.CUmemAccessDesc()
        acc.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = device
        acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc = ok(drv.cuMemAddressReserve(size, 0, 0, 0), "cuMemAddressReserve")
        ok(drv.cuMemMap(self.uc, size, 0, self.mem, 0), "cuMemMap")
        ok(drv.cuMemSetAccess(self.uc, size, [acc], 1), "cuMemSetAccess")
        self.mc = ok(drv.cuMemAddressReserve(size, 0, 0, 0), "cuMemAddressReserve")
        ok(drv.cuMemMap(self.mc, size, 0, self.mc_handle, 0), "cuMemMap")
        ok(drv.cuMemSetAccess(self.mc, size, [acc], 1), "cuMemSetAccess")

    def unicast_ptr(self) -> int:
        return int(self.uc)

    def multicast_ptr(self) -> int:
        return int(self.mc)

    def read(self, nbytes: int):
        """Copy the first nbytes (through the unicast mapping) into a host uint8 tensor."""
        torch.cuda.synchronize()
        out = torch.empty(nbytes, dtype=torch.uint8)
        res = self.drv.cuMemcpyDtoH(out.data_ptr(), self.uc, nbytes)
        err = res[0] if isinstance(res, tuple) else res
        if err != self.drv.CUresult.CUDA_SUCCESS:
            raise RuntimeError(f"cuMemcpyDtoH: {err}")
        return out

    def close(self):
        d = self.drv
        d.cuMemUnmap(self.mc, self.size)
        d.cuMemUnmap(self.uc, self.size)
        d.cuMemAddressFree(self.mc, self.size)
        d.cuMemAddressFree(self.uc, self.size)
        d.cuMulticastUnbind(self.mc_handle, 0, 0, self.size)
        d.cuMemRelease(self.mem)
        d.cuMemRelease(self.mc_handle)


def peer_ranks(rank: int, world: int):
    """The ranks whose C copies this rank writes besides its own (all others, in ring
    order starting after `rank` so the ranks' NVLink stores spread over destinations)."""
    return [(rank + d) % world for d in range(1, world)]
