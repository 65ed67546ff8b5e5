"""Multi-GPU sharding of the batch.

Realizations are independent (the reference's parallel_for treats them so,
parallel.hpp:12-18), so the batch shards with no data-path collective. Two
layouts are used:

* weak scaling (bench.py): rank r owns the global realizations
  [r*B, (r+1)*B) of a batch of world*B;
* strong scaling / the single-process sharded ABI: contiguous slices
  [g*B/G, (g+1)*B/G) of one fixed batch.

The only collective is the final reduction of the three summary statistics
(sum alpha*||W||_{2,1}, sum active, #diverged) — 24 bytes, one all-reduce.
"""
from __future__ import annotations

from typing import Tuple


def weak_shard(rank: int, per_rank: int) -> Tuple[int, int]:
    """(first global index, count) of a rank's realizations under weak scaling."""
    if rank < 0 or per_rank < 0:
        raise ValueError("rank and per_rank must be >= 0")
    return rank * per_rank, per_rank


def strong_shard(rank: int, world: int, total: int) -> Tuple[int, int]:
    """(first index, count) of contiguous slice `rank` of `total` over `world`
    ranks — the same split as ufpgd_gpu_unfolded_forward_sharded."""
    if not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard request")
    b0 = total * rank // world
    b1 = total * (rank + 1) // world
    return b0, b1 - b0


def reduce_stats(stats, group=None):
    """All-reduce (sum) of a rank's 3 statistics in place; a float64 tensor on
    the rank's device (NCCL) or the CPU (gloo). Returns the tensor."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def summarize(stats, total_realizations: int) -> dict:
    """Means of the reduced statistics (the north_star's mean consumed power
    and mean active-antenna count)."""
    s = [float(x) for x in stats]
    ok = total_realizations - s[2]
    return {"mean_consumed_power": s[0] / ok if ok > 0 else float("nan"),
            "mean_active": s[1] / ok if ok > 0 else float("nan"), "diverged": int(s[2])}
