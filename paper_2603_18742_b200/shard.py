"""Token sharding and the per-step statistics exchange.

Each rank owns a contiguous range of token rows; weights are replicated. Every
hot-path op is row-local, so the only communication is, once per timestep:
  - SUM all-reduce of a zero-padded [world x blocks x 11] FP64 slot buffer (each
    rank fills only its own slot: the SUM is an exact all-gather), then a
    rank-ordered combine, so every rank holds bit-identical global statistics;
  - MAX all-reduce of the [blocks x 8] fp32 activation maxima (NVFP4 global scales and
    the PDR outlier ratio's max|x|).
Works with any torch.distributed backend (NCCL on the GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np
import torch


def shard_rows(M: int, world: int, rank: int):
    """Contiguous row range [r0, r1) of `rank` (sizes differ by at most one)."""
    return (M * rank) // world, (M * (rank + 1)) // world


def exchange(stats_slots: torch.Tensor, amax: torch.Tensor, group=None, world: int = 1) -> np.ndarray:
    """All-reduce the slot-packed statistics (SUM) and the amax (MAX) in place and
    return the rank-order combined FP64 statistics [blocks x 7] on the host."""
    if group is not None and world > 1:
        torch.distributed.all_reduce(stats_slots, op=torch.distributed.ReduceOp.SUM, group=group)
        torch.distributed.all_reduce(amax, op=torch.distributed.ReduceOp.MAX, group=group)
    slots = stats_slots.cpu().numpy()
    out = np.zeros(slots.shape[1:], dtype=np.float64)
    for r in range(slots.shape[0]):
        out += slots[r]
    return out
