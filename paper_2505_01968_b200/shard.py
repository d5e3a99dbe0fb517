"""Sharding of the data-parallel work over one process per GPU (torch.distributed).

* Predictions (config 2): every rank owns its own query stream — replicas, no collective.
* Configuration search (config 5): contiguous blocks of functions per rank; each rank runs
  the fused lattice kernel on its block and ONE all-gather assembles the per-function
  (b, s, q) decisions in function order on every rank (NCCL over NVLink on B200; the same
  code runs on gloo for CPU tests).
* Ticks: the commit phase is an ordered scan over shared cluster state,
  so ticks run as replicas.
"""

from __future__ import annotations

import torch


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [begin, end) of n items owned by `rank` (balanced, in order)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return rank * n // world, (rank + 1) * n // world


def block_size(n: int, world: int) -> int:
    """Padded per-rank block length used by the all-gather (max shard size)."""
    return max(shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world))


def gather_decisions(local: torch.Tensor, n: int, world: int, group=None) -> torch.Tensor:
    """All-gather per-rank (rows, k) decision blocks into the (n, k) result in function
    order.  `local` must be padded to block_size(n, world) rows."""
    import torch.distributed as dist
    per = block_size(n, world)
    if local.shape[0] != per:
        raise ValueError(f"local block has {local.shape[0]} rows, expected {per}")
    if world == 1:
        return local[:n]
    full = torch.empty((per * world,) + tuple(local.shape[1:]), dtype=local.dtype,
                       device=local.device)
    dist.all_gather_into_tensor(full, local.contiguous(), group=group)
    parts = []
    for r in range(world):
        b, e = shard_range(n, r, world)
        parts.append(full[r * per: r * per + (e - b)])
    return torch.cat(parts, dim=0)


def search_sharded(table_set, targets: torch.Tensor, rank: int, world: int,
                   stream=None, group=None) -> torch.Tensor:
    """most_efficient_config for every function of a PerfTableSet, functions sharded over
    ranks: local fused lattice pass + one all-gather.  Returns (nfn, 3) int32 on device."""
    n = table_set.nfn
    b, e = shard_range(n, rank, world)
    per = block_size(n, world)
    local = torch.full((per, 3), -1, dtype=torch.int32, device=targets.device)
    table_set.search_dev(targets, local, fn_begin=b, fn_end=e, stream=stream)
    return gather_decisions(local, n, world, group=group)
