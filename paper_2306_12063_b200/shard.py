"""Codeword sharding across GPUs and the one collective the path has.

SURVEY.md §8e: codewords are independent, so a batch is split into contiguous
per-rank shards with no data-path exchange; the only collective is a final
sum of error / iteration counters (the multi-GPU analogue of the reference's
`run_waterfall` bookkeeping, `/root/reference/pkg/src/qcldpc/chansim.py:171-176`).
With one process per GPU, `torch.distributed` (NCCL on B200, gloo on CPU for
tests) carries that single all_reduce.
"""

from __future__ import annotations

COUNTERS = ("bit_errors", "frame_errors", "iter_sum", "converged", "frames")


def shard_range(w_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) of codewords owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world or w_total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(w_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def decode_counters(hard, iters, conv, ref_info, k: int):
    """int64[5] counters of one shard: bit errors / frame errors on the k
    systematic bits against the transmitted info, iteration sum, converged
    count, frames.  All tensors on the same device (torch)."""
    import torch
    err = (hard[:, :k] != ref_info[:, :k]).sum(dim=1)
    return torch.stack([err.sum(), (err > 0).sum(), iters.to(torch.int64).sum(),
                        conv.to(torch.int64).sum(),
                        torch.tensor(hard.shape[0], dtype=torch.int64, device=hard.device)])


def all_reduce_counters(cnt, group=None):
    """Sum the counter vector over ranks (one collective; no-op when not distributed)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
    return cnt
