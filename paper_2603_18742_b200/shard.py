"""Token sharding and the per-step statistics exchange.

Each rank owns a contiguous range of token rows; weights are replicated. Every
hot-path op is row-local, so the only communication is ONE collective per
timestep: a SUM all-reduce of a zero-padded FP64 slot buffer [world x (S + A)],
in which each rank fills only its own slot with
  - its S FP64 partial statistics (7 TDC/predictor sums + PDR sums per block), and
  - its A fp32 maxima (activation amax for the NVFP4 global scales, PDR max|x|,
    delta-cache amax), widened to FP64 (exact).
Adding zeros is exact, so the SUM is an all-gather: afterwards every rank
combines the statistics in rank order (bit-identical on every rank) and takes
the maximum over the slots' maxima (exact). The collective's payload is ~4 KB
for CogVideoX-5B (42 blocks). Works with any torch.distributed backend (NCCL on
the GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np
import torch


def shard_rows(M: int, world: int, rank: int):
    """Contiguous row range [r0, r1) of `rank` (sizes differ by at most one)."""
    return (M * rank) // world, (M * (rank + 1)) // world


class SlotBuffer:
    """The per-step exchange buffer [world x (n_stats + n_max)] (FP64, zero-initialised).

    stats  -- [world x n_stats] view; a rank's kernels write its partial sums into stats[rank]
    maxima -- [world x n_max] view; filled from the rank's fp32 maxima by pack_maxima()."""

    def __init__(self, world: int, rank: int, n_stats: int, n_max: int, device):
        self.world, self.rank, self.n_stats, self.n_max = world, rank, n_stats, n_max
        self.buf = torch.zeros(world, n_stats + n_max, dtype=torch.float64, device=device)
        self.stats = self.buf[:, :n_stats]
        self.maxima = self.buf[:, n_stats:]

    def zero_(self):
        self.buf.zero_()

    def pack_maxima(self, amax: torch.Tensor):
        """This rank's fp32 maxima (non-negative) into its slot, widened to FP64 (exact)."""
        self.maxima[self.rank].copy_(amax.reshape(-1))


def exchange_device(slots: SlotBuffer, amax: torch.Tensor | None = None, group=None) -> None:
    """One SUM all-reduce of the slot buffer (an exact all-gather), then amax <- the maximum over
    the ranks' slots, in place (fp32; exact: the values are fp32). Enqueued on the current stream."""
    if group is None or slots.world == 1:
        return
    if amax is not None:
        slots.pack_maxima(amax)
    torch.distributed.all_reduce(slots.buf, op=torch.distributed.ReduceOp.SUM, group=group)
    if amax is not None:
        amax.reshape(-1).copy_(slots.maxima.max(dim=0).values)


def combine_host(slots: SlotBuffer) -> np.ndarray:
    """The rank-order combined FP64 statistics [n_stats] on the host (the D2H copy synchronises
    the stream); bit-identical on every rank."""
    host = slots.stats.cpu().numpy()
    out = np.zeros(slots.n_stats, dtype=np.float64)
    for r in range(slots.world):
        out += host[r]
    return out


def exchange(slots: SlotBuffer, amax: torch.Tensor | None = None, group=None) -> np.ndarray:
    """exchange_device + combine_host."""
    exchange_device(slots, amax, group)
    return combine_host(slots)
