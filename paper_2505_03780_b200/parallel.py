"""Multi-GPU plumbing for the attention hot path.

The path shards with no exchange step: every (sequence, kv-head group) is independent, so the
8 B200s of a box each take a contiguous shard of the batch (decode: C4's 256 sequences -> 32 per
GPU, each GPU holding only its sequences' pages) or of the kv-head groups (prefill), and run the
same kernels with no cross-GPU reduction.  torch.distributed (NCCL on GPUs, gloo on CPU) is used
only for barriers, the max-over-ranks of the timed region, and gathering outputs to rank 0 for
validation against the CPU oracle — never inside the timed region.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Shard:
    start: int
    count: int


def shard_range(total: int, world: int, rank: int) -> Shard:
    """Contiguous, balanced split of `total` units (sizes differ by at most one)."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return Shard(start, base + (1 if rank < extra else 0))


def kv_head_groups(num_kv_heads: int, world: int, rank: int) -> range:
    """Prefill sharding by GQA group: each rank owns whole kv heads (and their q heads)."""
    s = shard_range(num_kv_heads, world, rank)
    return range(s.start, s.start + s.count)


def env_world():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(
        os.environ.get("LOCAL_RANK", "0"))


def max_over_ranks(x: float) -> float:
    """Timed regions are reported as the slowest rank's time."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_rank0(t: torch.Tensor, counts: list[int]):
    """Validation only: concatenate each rank's leading-dim shard on rank 0 (None elsewhere)."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return t
    world, rank = dist.get_world_size(), dist.get_rank()
    pad = max(counts)
    dev = t.device if dist.get_backend() == "nccl" else torch.device("cpu")  # gloo gathers host tensors
    buf = torch.zeros((pad,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
    buf[: t.shape[0]] = t.to(dev)
    bufs = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, bufs, dst=0)
    if rank != 0:
        return None
    return torch.cat([b[:c] for b, c in zip(bufs, counts)])


def weak_scaling_value(units_per_rank: float, steps: int, ms_max: float, world: int, scale: float) -> float:
    """Whole-job throughput: units processed by all ranks / slowest rank's time."""
    return world * units_per_rank * steps / (ms_max / 1e3) / scale
