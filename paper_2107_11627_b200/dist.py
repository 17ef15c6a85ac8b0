"""Multi-GPU plumbing for the batch-sharded render.

Frames are independent (PAPER.md:474 sequences; temporal correlation is out of scope), so N
GPUs render disjoint frames with replicated basis/weights and no collective on the data
path ("scaling": "weak"). The only collectives are the timing barrier and the max-over-ranks
reduction of the measured time. One process per GPU, torch.distributed (NCCL on GPUs, gloo in
the CPU tests).
"""
from __future__ import annotations

import os
from typing import Optional


def env_rank_world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def rank_frames(rank: int, frames_per_rank: int) -> range:
    """Frame indices (seeds) rendered by `rank`: a contiguous, disjoint block per rank."""
    if rank < 0 or frames_per_rank < 1:
        raise ValueError("rank must be >= 0 and frames_per_rank >= 1")
    return range(rank * frames_per_rank, (rank + 1) * frames_per_rank)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (e.g. elapsed ms) over all ranks; identity without a group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def throughput(frames_per_rank: int, world: int, steps: int, max_ms: float) -> float:
    """Whole-job frames/s: every rank's frames over the slowest rank's time."""
    if max_ms <= 0:
        raise ValueError("time must be positive")
    return frames_per_rank * world * steps / (max_ms / 1e3)


def init(backend: str, device_id=None):
    """init_process_group from the torchrun env (MASTER_ADDR/PORT); returns the dist module."""
    import torch.distributed as dist
    if not dist.is_initialized():
        kw = {"device_id": device_id} if device_id is not None else {}
        dist.init_process_group(backend, **kw)
    return dist


def shutdown(dist) -> None:
    if dist is not None and dist.is_initialized():
        dist.destroy_process_group()
