"""world_size-2 gloo tests of the sharded configuration search (CPU).

Each rank computes its contiguous block of most_efficient_config decisions (here with
the CPU oracle standing in for the device kernel, which needs a GPU) and the product's
gather_decisions assembles them; the result must equal the single-process answer in
function order, for function counts that do and do not divide evenly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_01968_b200.shard import block_size, gather_decisions, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _tables(n):
    rng = np.random.default_rng(5)
    out = []
    for i in range(n):
        fixed, per, floor = rng.uniform(4, 20), rng.uniform(0.5, 4), rng.uniform(0.2, 0.4)
        b = np.array([1.0, 2.0, 4.0, 8.0])
        s = np.arange(10.0, 101.0, 10.0)
        q = np.arange(10.0, 101.0, 10.0)
        v = ((fixed + per * b)[:, None, None] * (floor + (1 - floor) * (100.0 / s))[None, :, None]
             * (100.0 / q)[None, None, :])
        out.append((b, s, q, np.ascontiguousarray(v), float(rng.uniform(5, 400))))
    return out


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.binding import or_most_efficient_config
    tabs = _tables(n)
    b0, e0 = shard_range(n, rank, world)
    per = block_size(n, world)
    local = torch.full((per, 3), -1, dtype=torch.int32)
    for i, f in enumerate(range(b0, e0)):
        b, s, qq, v, target = tabs[f]
        local[i] = torch.tensor(or_most_efficient_config(b, s, qq, v, target, 10, None))
    full = gather_decisions(local, n, world)
    q.put((rank, full.numpy().tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 8, 1])
def test_gloo_world2_sharded_search_matches_single_process(n):
    from oracle.binding import or_most_efficient_config
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [list(or_most_efficient_config(b, s, qq, v, t, 10, None))
            for b, s, qq, v, t in _tables(n)]
    assert results[0] == want and results[1] == want


def test_shard_ranges_cover_in_order():
    for n in (0, 1, 5, 3125):
        for world in (1, 2, 4, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - b for b, e in spans) == block_size(n, world) or n == 0
