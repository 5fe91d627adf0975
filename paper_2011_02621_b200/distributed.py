"""Multi-GPU sharding of amplitude evaluation (one process per GPU).

The work of a batched evaluation is the grid of independent items
(bitstring b, slice s), b < B, s < S.  Items are flattened bitstring-major and
split into W contiguous ranges, one per rank, so each rank contracts whole
bitstrings where B >= W and slice ranges of a bitstring otherwise -- no data
moves between GPUs while contracting.  Each rank accumulates its partial slice
sums into a length-B amplitude vector (zeros elsewhere); a single NCCL
all-reduce (sum) then performs the slice-sum and the amplitude gather at once
(the reference's slice loop, network.py:334-339, distributed).
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["WorkRange", "shard_items", "rank_chunks", "run_sharded", "sharded_amplitudes"]


@dataclass(frozen=True)
class WorkRange:
    """Bitstrings [b0, b0 + nb) over slices [s0, s1) (a rectangular chunk)."""

    b0: int
    nb: int
    s0: int
    s1: int


def shard_items(B: int, S: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous flattened item range [i0, i1) of ``rank``."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    total = B * S
    return rank * total // world, (rank + 1) * total // world


def rank_chunks(B: int, S: int, rank: int, world: int) -> list[WorkRange]:
    """The rank's item range as at most three rectangular chunks: a partial
    bitstring tail, a block of whole bitstrings, a partial bitstring head."""
    i0, i1 = shard_items(B, S, rank, world)
    out: list[WorkRange] = []
    if i0 >= i1:
        return out
    b_first, s_first = divmod(i0, S)
    b_last, s_last = divmod(i1, S)          # exclusive end
    if b_first == b_last:
        return [WorkRange(b_first, 1, s_first, s_last)]
    b = b_first
    if s_first:
        out.append(WorkRange(b_first, 1, s_first, S))
        b += 1
    if b_last > b:
        out.append(WorkRange(b, b_last - b, 0, S))
    if s_last:
        out.append(WorkRange(b_last, 1, 0, s_last))
    return out


def run_sharded(executor, sel, B: int, amp, rank: int, world: int) -> None:
    """Contract this rank's share into ``amp`` (zero-initialised, length B).
    ``executor.run(sel, nb, amp, slices=range, b_offset=b0, accumulate=True)``."""
    S = executor.plan.slice_count
    for ch in rank_chunks(B, S, rank, world):
        executor.run(sel, ch.nb, amp, slices=range(ch.s0, ch.s1), b_offset=ch.b0, accumulate=True)


def sharded_amplitudes(executor, sel, B: int, amp, group=None):
    """run_sharded + one all-reduce(sum): slice-sum and amplitude gather."""
    import torch.distributed as dist

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    amp.zero_()
    run_sharded(executor, sel, B, amp, rank, world)
    if world > 1:
        dist.all_reduce(amp, op=dist.ReduceOp.SUM, group=group)
    return amp
