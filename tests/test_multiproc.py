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


# -- the product's sharding entry points, driven by oracle-backed stand-ins ------------------

class _OracleTable:
    """A PerfTable stand-in for CPU tests: the C oracle answers most_efficient_config and
    throughput (the device kernels need a GPU); the product's shard.search_split does the
    slab split, key packing and collectives."""

    def __init__(self, b, s, q, v):
        self._b_axis, self._s_axis, self._q_axis, self.latency_ms = b, s, q, v
        self.batches = [int(x) for x in b]
        self.sms = [int(x) for x in s]

    def _batch_lattice(self, batches):
        if batches is not None:
            inside = {int(x) for x in batches if self.batches[0] <= x <= self.batches[-1]}
            if inside:
                return sorted(inside)
        return list(self.batches)

    def most_efficient_config(self, target, *, quota_step=10, batches=None):
        from oracle.binding import or_most_efficient_config
        return tuple(or_most_efficient_config(self._b_axis, self._s_axis, self._q_axis,
                                              self.latency_ms, target, quota_step,
                                              self._batch_lattice(batches)))

    def throughput(self, b, s, q):
        from oracle.binding import or_interp3, or_throughput
        return or_throughput(float(b), or_interp3(self._b_axis, self._s_axis, self._q_axis,
                                                  self.latency_ms, float(b), float(s), float(q)))


class _OracleSet:
    """PerfTableSet stand-in: search_dev fills (b, s, q) rows of [fn_begin, fn_end)."""

    def __init__(self, tabs, step):
        self.tabs, self.step, self.nfn = tabs, step, len(tabs)

    def search_dev(self, targets, out, fn_begin=0, fn_end=None, stream=None):
        from oracle.binding import or_most_efficient_config
        for i, f in enumerate(range(fn_begin, fn_end)):
            b, s, q, v, _ = self.tabs[f]
            out[i] = torch.tensor(or_most_efficient_config(b, s, q, v, float(targets[f]),
                                                           self.step, None))
        return out


def _big_table():
    rng = np.random.default_rng(11)
    b = np.arange(1.0, 33.0)
    s = np.arange(10.0, 101.0, 10.0)
    q = np.arange(10.0, 101.0, 10.0)
    v = ((6.0 + 1.7 * b)[:, None, None] * (0.3 + 0.7 * (100.0 / s))[None, :, None]
         * (100.0 / q)[None, None, :]) * (1.0 + 0.01 * rng.random((len(b), len(s), len(q))))
    return _OracleTable(b, s, q, np.ascontiguousarray(v))


SPLIT_CASES = [(5.0, 10, None), (300.0, 10, None), (900.0, 5, [2, 3, 5, 7, 11, 13, 30]),
               (1e9, 10, None), (1e9, 20, [4, 8]), (40.0, 1, [1])]


def _product_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_01968_b200.shard import search_sharded, search_split
    tabs = _tables(7)
    targets = torch.tensor([t[4] for t in tabs], dtype=torch.float64)
    full = search_sharded(_OracleSet(tabs, 10), targets, rank, world)
    big = _big_table()
    split = [search_split(big, t, rank, world, quota_step=st, batches=bl)
             for t, st, bl in SPLIT_CASES]
    q.put((rank, full.numpy().tolist(), split))
    dist.destroy_process_group()


def test_gloo_world2_product_sharding_entry_points():
    """shard.search_sharded over a (stand-in) PerfTableSet and shard.search_split of one
    lattice over batch slabs — meet by all-reduce MIN, fallback by all-gather — equal the
    single-process most_efficient_config on both ranks."""
    from oracle.binding import or_most_efficient_config
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_product_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict((r, (a, b)) for r, a, b in (q.get(timeout=180) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [list(or_most_efficient_config(b, s, qq, v, t, 10, None))
            for b, s, qq, v, t in _tables(7)]
    big = _big_table()
    want_split = [tuple(big.most_efficient_config(t, quota_step=st, batches=bl))
                  for t, st, bl in SPLIT_CASES]
    for r in range(world):
        assert results[r][0] == want
        assert [tuple(x) for x in results[r][1]] == want_split


def test_split_single_rank_matches():
    from paper_2505_01968_b200.shard import search_split
    big = _big_table()
    for t, st, bl in SPLIT_CASES:
        assert search_split(big, t, 0, 1, quota_step=st, batches=bl) == \
            tuple(big.most_efficient_config(t, quota_step=st, batches=bl))


def test_bench_self_launches_n_ranks_on_cpu():
    """`bench.py --gpus 2` outside torchrun relaunches itself as 2 ranks through
    torch.distributed.run (127.0.0.1); the reference arm needs no GPU, so the whole path —
    launch, rank 0 alone printing one JSON line with n_gpus = 2, rank 1 exiting 0 — runs on
    CPU.  Needs the reference kernel built by build() (oracle/_ref)."""
    import glob
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if not glob.glob(os.path.join(root, "oracle", "_ref", "_grid_cy*.so")):
        pytest.skip("oracle/_ref not built (run build())")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["impl"] == "reference" and line["value"] > 0
