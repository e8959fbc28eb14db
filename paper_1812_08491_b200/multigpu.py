"""Multi-GPU PC-stable: one process per GPU, per-level sharding, one MIN all-reduce
of the level's key array after each pass.

Every rank holds the replicated correlation matrix and builds the identical
snapshot; pass p of a level is split into contiguous work-unit ranges (rank r
of N takes units [r*U/N, (r+1)*U/N)).  A key is (dir << 62 | rank of the first
separating set) per undirected edge, so MIN over ranks is exactly the serial
strategy's choice and subsumes the "bitwise AND of the live mask" merge (NCCL
has no AND).  The commit that follows is replicated and deterministic.

The level loop is written against a small protocol (level_begin / level_pass /
keys / level_end / finish) so the same orchestration is exercised on CPU with
gloo and an oracle-backed session in tests/test_multigpu_gloo.py.
"""
from __future__ import annotations

from typing import Callable, Optional


def level_loop(session, allreduce_min: Optional[Callable[[object, int], None]], world: int):
    """Runs the PC-stable level loop on `session`; `allreduce_min(ptr_or_array, n)` merges keys."""
    while True:
        running, ell, nkeys = session.level_begin()
        if not running:
            break
        passes = session.level_passes() if hasattr(session, "level_passes") else 2
        for pass_index in (0, 1):
            session.level_pass(pass_index)
            if pass_index < passes and world > 1 and nkeys > 0 and allreduce_min is not None:
                keys, n = session.keys()
                allreduce_min(keys, n)
        session.level_end()
    return session


class _CudaArray:
    """__cuda_array_interface__ view of library-owned device memory (int64 keys)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False), "version": 3,
                                         "strides": None}


def torch_allreduce_min(group=None):
    """MIN all-reduce of a device key array through torch.distributed (NCCL over NVLink)."""
    import torch
    import torch.distributed as dist

    def _reduce(ptr: int, n: int):
        t = torch.as_tensor(_CudaArray(ptr, n), device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        torch.cuda.current_stream().synchronize()

    return _reduce


def host_staged_allreduce_min(group=None):
    """MIN all-reduce through host memory (gloo): ranks sharing one GPU in tests, or any transport
    without device-buffer support.  Same result as torch_allreduce_min."""
    import torch
    import torch.distributed as dist

    def _reduce(ptr: int, n: int):
        dev = torch.as_tensor(_CudaArray(ptr, n), device="cuda")
        host = dev.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.MIN, group=group)
        dev.copy_(host)
        torch.cuda.current_stream().synchronize()

    return _reduce


def row_band(p: int, rank: int, world: int) -> tuple[int, int, int]:
    """(row_begin, row_end, band) of this rank's correlation rows: equal bands of ceil(p / world) rows
    (all_gather_into_tensor needs equal chunks; the last band may be short or empty)."""
    band = (p + world - 1) // world
    r0 = min(p, rank * band)
    return r0, min(p, r0 + band), band


def correlation_sharded(x_ptr: int, m: int, p: int, c, group=None, stream: int = 0, gather=None):
    """compute_correlation split over the ranks: rank r builds rows
    [r * B, (r + 1) * B) of C (B = ceil(p / N)) with its own Gram row band, then the bands are
    all-gathered into every rank's copy (NCCL over NVLink by default).  `c` is a torch float64 tensor
    of shape (N * B, ldc) on this rank's device; rows >= p are scratch.  The assembled rows are
    bit-identical to a one-GPU correlation_device (tests/test_gpu_multiproc.py)."""
    import torch
    import torch.distributed as dist

    from . import correlation_device_rows

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    r0, r1, band = row_band(p, rank, world)
    ldc = c.shape[1]
    assert c.shape[0] >= band * world and c.dtype == torch.float64
    correlation_device_rows(x_ptr, m, p, r0, r1, c.data_ptr(), ldc, stream)
    if world > 1:
        torch.cuda.synchronize()
        mine = c[rank * band:(rank + 1) * band].clone()
        (gather or dist.all_gather_into_tensor)(c[:band * world], mine, group=group)
        torch.cuda.synchronize()
    return c


def host_staged_all_gather(out, inp, group=None):
    """all_gather_into_tensor through host memory (gloo: ranks sharing one GPU in tests)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    parts = [torch.empty_like(inp, device="cpu") for _ in range(world)]
    dist.all_gather(parts, inp.cpu(), group=group)
    out.copy_(torch.cat(parts).to(out.device))


def run_pc_stable_sharded(c_ptr: int, ldc: int, p: int, sample_count: int, cfg=None, group=None,
                          with_sepsets: bool = True, allreduce_min=None):
    """run_pc_stable over all ranks of `group` (torch.distributed initialised, one GPU per rank).
    allreduce_min: key reducer (default: NCCL on the device buffers)."""
    import torch.distributed as dist

    from . import Session, SkeletonConfig

    cfg = cfg or SkeletonConfig()
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    s = Session(sample_count=sample_count, cfg=cfg, shard_index=rank, shard_count=world, device_ptr=c_ptr, ldc=ldc,
                p=p)
    try:
        red = allreduce_min or torch_allreduce_min(group)
        level_loop(s, red if world > 1 else None, world)
        return s.finish(with_sepsets)
    finally:
        s.close()
