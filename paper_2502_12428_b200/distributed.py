"""Multi-GPU sharding of a batch: one process per GPU (torch.distributed), no data-path collective.

Surfaces are independent, so rank r computes the r-th contiguous block of the
batch -- the reference's worker partition (search.py:128-135) with worker = rank -- and the only
communication is the final gather of one int8 height and one int8 iteration count per surface
(`torch.distributed.all_gather` on the process group's backend: NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np

from .height import split_blocks


def rank_block(total: int, rank: int, world: int):
    """(start, count) of rank's block; ranks beyond the batch size get an empty block."""
    blocks = split_blocks(total, world)
    return blocks[rank] if rank < len(blocks) else (total, 0)


def heights_sharded(p: int, coeffs, bound: int = 10, device=None, group=None, compute=None, method: str = "matrix"):
    """Heights of the global batch `coeffs` [B,35] (same array on every rank), computed block-wise.

    Every rank returns the full (heights int8[B], iterations int8[B]).  `device`: CUDA device index of this
    rank (default: rank % device_count); `compute(p, coeffs, bound, device)` replaces the CUDA engine in
    CPU tests; `method` as in height_batch ("matrix", "lazy", "naive").
    """
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    c = np.ascontiguousarray(coeffs, dtype=np.uint8)
    B = c.shape[0]
    start, count = rank_block(B, rank, world)
    if compute is None:
        from .height import height_batch
        dev = device if device is not None else rank % max(1, torch.cuda.device_count())
        hs, its = height_batch(p, c[start:start + count], bound, devices=[dev], method=method) if count else (np.empty(0, np.int8),) * 2
    else:
        hs, its = compute(p, c[start:start + count], bound, device) if count else (np.empty(0, np.int8),) * 2
    if world == 1:
        return np.asarray(hs, np.int8), np.asarray(its, np.int8)
    use_cuda = dist.get_backend(group) == "nccl"
    tdev = torch.device("cuda", torch.cuda.current_device()) if use_cuda else torch.device("cpu")
    width = max(n for _, n in split_blocks(B, world))
    mine = torch.zeros(2, width, dtype=torch.int8, device=tdev)
    mine[0, :count] = torch.from_numpy(np.asarray(hs, np.int8)).to(tdev)
    mine[1, :count] = torch.from_numpy(np.asarray(its, np.int8)).to(tdev)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    heights = np.empty(B, np.int8)
    iters = np.empty(B, np.int8)
    for r in range(world):
        s, n = rank_block(B, r, world)
        blk = parts[r].cpu().numpy()
        heights[s:s + n] = blk[0, :n]
        iters[s:s + n] = blk[1, :n]
    return heights, iters
