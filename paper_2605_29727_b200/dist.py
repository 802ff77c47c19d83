"""Multi-GPU plumbing for decode: one process per GPU, independent requests, no
collective on the data path.  Only the bench's timing uses a
collective: the max of the per-rank device-timed regions and the sum of the
committed tokens (whole-job throughput = total tokens / slowest rank)."""

from __future__ import annotations

import os

import torch


def world() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_requests: int, world_size: int, rank: int) -> range:
    """Contiguous request shard of this rank (config 3: 64 requests over 1/2/4/8 GPUs)."""
    if n_requests < 0 or world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n_requests, world_size)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def reduce_throughput(elapsed_s: float, tokens: float, device=None) -> tuple[float, float, float]:
    """(max elapsed over ranks, total tokens, tokens/s) — identity when not distributed."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return elapsed_s, tokens, tokens / elapsed_s
    dev = device if device is not None else ("cuda" if dist.get_backend() == "nccl" else "cpu")
    mx = torch.tensor([elapsed_s], dtype=torch.float64, device=dev)
    sm = torch.tensor([tokens], dtype=torch.float64, device=dev)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return float(mx.item()), float(sm.item()), float(sm.item()) / float(mx.item())
