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
    ranks: local fused lattice pass + one all-gather.  Returns (nfn, 3) int32 on device.
    `table_set` is anything with `nfn` and `search_dev(targets, out, fn_begin=, fn_end=,
    stream=)` (the CPU tests drive it with an oracle-backed stand-in)."""
    n = table_set.nfn
    b, e = shard_range(n, rank, world)
    per = block_size(n, world)
    local = torch.full((per, 3), -1, dtype=torch.int32, device=targets.device)
    table_set.search_dev(targets, local, fn_begin=b, fn_end=e, stream=stream)
    return gather_decisions(local, n, world, group=group)


# -- one giant lattice split over ranks (contiguous batch slabs) ------------

NO_KEY = (1 << 63) - 1


def pack_key(s_idx: int, s: int, q: int, b_idx: int) -> int:
    """The search's total order (s*q, s, q, b) as one integer — the packing of the lattice
    kernel (rapp_search.cu: cost << 32 | s_idx << 20 | q << 12 | b_idx) with b_idx the
    index in the WHOLE batch lattice, so keys of different slabs compare correctly."""
    return (s * q) << 32 | s_idx << 20 | q << 12 | b_idx


def search_split(table, target_rps: float, rank: int, world: int, *, quota_step: int = 10,
                 batches=None, group=None) -> tuple[int, int, int]:
    """most_efficient_config (hs/perf.py:104-145) of ONE table whose lattice is split over
    ranks by contiguous slabs of its batch lattice (`_batch_lattice` rule, perf.py:140-145).

    Each rank searches its slab on its own device (`table.most_efficient_config` restricted
    to the slab), then:
      * meet: one all-reduce MIN of the packed (s*q, s, q, b) key of the slab's feasible
        answer (NO_KEY when the slab has none) — the common case, one collective;
      * fallback, only when no slab meets the target: one all-gather of 16-byte records
        (order-preserving bits of the slab's max rps, its packed key) reduced locally to
        max rps, then min key — the reference's argmin (-rps, s*q, s, q, b).
    Every rank returns the same (b, s, q).  `table` is a PerfTable (or anything with
    `_batch_lattice`, `sms`, `most_efficient_config`, `throughput`)."""
    import struct
    import torch.distributed as dist
    if target_rps <= 0:
        raise ValueError("target_rps must be positive")
    if not 1 <= quota_step <= 100:
        raise ValueError("quota_step must be in [1, 100]")
    lattice = list(table._batch_lattice(batches))
    b0, b1 = shard_range(len(lattice), rank, world)
    key, rps_bits = NO_KEY, -1
    meet = False
    if b1 > b0:
        slab = lattice[b0:b1]
        b, s, q = table.most_efficient_config(target_rps, quota_step=quota_step, batches=slab)
        rps = float(table.throughput(b, s, q))
        meet = rps >= target_rps
        key = pack_key(list(table.sms).index(s), s, q, lattice.index(b))
        rps_bits = struct.unpack("<q", struct.pack("<d", rps))[0]  # rps > 0: order-preserving
    if world == 1:
        return _decode(table, lattice, key)
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = torch.tensor([key if meet else NO_KEY], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    best = int(t.item())
    if best != NO_KEY:
        return _decode(table, lattice, best)
    mine = torch.tensor([rps_bits, key], dtype=torch.int64, device=dev)
    allrec = torch.empty(2 * world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allrec, mine, group=group)
    recs = [tuple(r) for r in allrec.view(world, 2).cpu().tolist()]
    top = max(r[0] for r in recs)
    return _decode(table, lattice, min(r[1] for r in recs if r[0] == top))


def _decode(table, lattice, key: int) -> tuple[int, int, int]:
    return (int(lattice[key & 0xFFF]), int(list(table.sms)[(key >> 20) & 0xFFF]),
            int((key >> 12) & 0xFF))
