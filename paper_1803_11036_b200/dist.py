"""Multi-router operation: one process per GPU (router), torch.distributed for
the plumbing (reference run_detection's merge branch,
pipeline.cpp:76-85, and merge_rseas, snapshot.cpp:117-142).

Union-min (the reference default) is idempotent and commutes with
advance_slot, so every router can keep the *merged* grid: in lockstep the
merged grid changes per slot exactly by "stamp = now on every recorder any
router touched".  The exchange is therefore the slot's touched bitmap (1 bit
per recorder, 1/32 of the stamp grid), OR-reduced across routers, then folded
into each router's stamps by the same commit kernel a single router uses.  The
result equals merge_rseas(node grids, kUnionMin) of the reference bit for bit
(tests/test_dist_gloo.py on CPU, tests/test_gpu_parity.py on the device).

paper-max keeps per-node grids and needs the full stamps: element-wise MIN
into a scratch copy (out of place, or it would corrupt later slots).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def or_allreduce_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place bitwise-OR all-reduce of an int32 tensor (NCCL has no OR op).

    Reduce-scatter by all_to_all + a local OR of the received chunks, then
    all-gather: the 2(N-1)/N per-rank volume of a ring all-reduce.  The same
    code runs on NCCL (GPU) and gloo (the CPU tests).
    """
    world = dist.get_world_size(group)
    if world == 1:
        return t
    flat = t.view(-1)
    n = flat.numel()
    per = (n + world - 1) // world
    padded = flat
    if per * world != n:
        padded = torch.zeros(per * world, dtype=flat.dtype, device=flat.device)
        padded[:n].copy_(flat)
    recv = torch.empty_like(padded)
    dist.all_to_all_single(recv, padded, group=group)
    chunks = recv.view(world, per)
    mine = chunks[0].clone()
    for i in range(1, world):
        mine.bitwise_or_(chunks[i])
    out = torch.empty_like(padded)
    dist.all_gather_into_tensor(out, mine, group=group)
    flat.copy_(out[:n])
    return t


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory owned by the grid."""

    def __init__(self, ptr: int, n: int, typestr: str = "<i4"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def device_view(ptr: int, n_words: int, device: int) -> torch.Tensor:
    with torch.cuda.device(device):
        return torch.as_tensor(_CudaArray(ptr, n_words), device=f"cuda:{device}")


def prepare(grid):
    """Make the grid record each slot's touched bitmap (needed in direct mode)."""
    grid.set_exchange(True)


def merge_touched(grid, group=None):
    """Union-min merge of this slot's touches across routers (in place)."""
    ptr, n = grid.touched_ptr()
    bits = device_view(ptr, n, grid.device)
    or_allreduce_(bits, group)
    torch.cuda.synchronize(grid.device)  # the grid's stream may differ from torch's
    grid.commit()


def merge_stamps_max(grid, group=None):
    """The literal north-star merge: all-reduce(max) of the full stamp grid.
    Correct but moves 32x the bytes of merge_touched; kept for comparison."""
    ptr, n = grid.stamps_ptr()
    st = device_view(ptr, n, grid.device)
    dist.all_reduce(st, op=dist.ReduceOp.MAX, group=group)
