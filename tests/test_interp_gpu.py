"""K2 stream interpolation on the B200 vs the reference's golden vectors and the oracle
(0-ulp).  Mirrors pkg/tests/test_kernels.py and the interpolation half of test_perf.py."""

import math
import random

import numpy as np
import pytest

from oracle.binding import or_interp3_many, or_locate, or_throughput

from .conftest import fromhex, golden_table_arrays, same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kern():
    from paper_2505_01968_b200 import kernels
    return kernels


def test_golden_vectors_bit_exact(kern, interp_golden):
    for rec in interp_golden["tables"]:
        b, s, q, v = golden_table_arrays(rec["table"])
        coords = fromhex(rec["coords"]).reshape(-1, 3)
        out = np.empty(len(coords))
        kern.interp3_many(b, s, q, v, coords, out)
        assert same_bits(out, fromhex(rec["latency"])), rec["table"]["function_id"]


def test_locate_golden(kern, interp_golden):
    for rec in interp_golden["locate"]:
        lo, hi, t = kern.locate(fromhex(rec["axis"]), float.fromhex(rec["x"]))
        want = float.fromhex(rec["t"])
        assert (lo, hi) == (rec["lo"], rec["hi"])
        assert (math.isnan(t) and math.isnan(want)) or t == want


def _grid():
    # pkg/tests/test_kernels.py:12-19
    b = np.array([1.0, 2.0, 4.0, 8.0])
    s = np.array([25.0, 50.0, 75.0, 100.0])
    q = np.array([10.0, 40.0, 70.0, 100.0])
    rng = random.Random(7)
    v = np.array([[[10.0 + 5 * bi + 2 * (3 - si) + (3 - qi) + rng.random()
                    for qi in range(4)] for si in range(4)] for bi in range(4)])
    return b, s, q, np.ascontiguousarray(v)


def test_exact_at_every_node(kern):
    b, s, q, v = _grid()
    for bi, bv in enumerate(b):
        for si, sv in enumerate(s):
            for qi, qv in enumerate(q):
                assert kern.interp3(b, s, q, v, bv, sv, qv) == v[bi, si, qi]


def test_quota_midpoint_and_clamps(kern):
    assert kern.interp3(np.array([1.0]), np.array([50.0]), np.array([20.0, 40.0]),
                        np.array([[[20.0, 30.0]]]), 1.0, 50.0, 30.0) == 25.0
    b, s, q, v = _grid()
    assert kern.interp3(b, s, q, v, 1.0, 5.0, 50.0) == kern.interp3(b, s, q, v, 1.0, 25.0, 50.0)
    assert kern.interp3(b, s, q, v, 1.0, 50.0, 300.0) == kern.interp3(b, s, q, v, 1.0, 50.0, 100.0)


@pytest.mark.parametrize("shape", [(4, 4, 10), (6, 10, 10), (6, 100, 100), (1, 1, 1),
                                   (1, 3, 2), (32, 91, 100)])
def test_random_coords_match_oracle(kern, shape):
    nb, ns, nq = shape
    rng = np.random.default_rng(sum(shape))
    b = np.cumsum(rng.uniform(0.5, 3, nb))
    s = np.cumsum(rng.uniform(0.5, 3, ns))
    q = np.cumsum(rng.uniform(0.5, 3, nq))
    v = np.ascontiguousarray(rng.uniform(1, 1000, shape))
    n = 200_003
    c = np.column_stack([rng.uniform(b[0] - 1, b[-1] + 1, n), rng.uniform(s[0] - 1, s[-1] + 1, n),
                         rng.uniform(q[0] - 1, q[-1] + 1, n)])
    c[::5, 0] = rng.choice(b, len(c[::5]))
    c[1::5, 1] = rng.choice(s, len(c[1::5]))
    c[2::5, 2] = rng.choice(q, len(c[2::5]))
    c[3] = [np.nan, s[0], q[0]]
    out = np.empty(n)
    kern.interp3_many(b, s, q, v, c, out)
    assert same_bits(out, or_interp3_many(b, s, q, v, c))


def test_empty_and_pinned_multi_chunk(kern):
    import torch
    b, s, q, v = _grid()
    out = np.empty(0)
    kern.interp3_many(b, s, q, v, np.empty((0, 3)), out)
    n = (1 << 21) * 2 + 12345  # three pipeline chunks
    rng = np.random.default_rng(3)
    c = np.column_stack([rng.uniform(0, 9, n), rng.uniform(20, 105, n), rng.uniform(5, 105, n)])
    want = or_interp3_many(b, s, q, v, c)
    got = np.empty(n)
    kern.interp3_many(b, s, q, v, c, got)  # pageable path
    assert same_bits(got, want)
    pc = torch.from_numpy(c).pin_memory()
    po = torch.empty(n, dtype=torch.float64).pin_memory()
    kern.interp3_many(b, s, q, v, pc.numpy(), po.numpy())  # pinned DMA path
    assert same_bits(po.numpy(), want)


def test_perftable_device_api_latency_and_rps():
    import torch
    from paper_2505_01968_b200 import PerfTable
    rng = np.random.default_rng(11)
    lat = np.sort(rng.uniform(1, 50, (6, 10, 10)), axis=0)[:, ::-1, ::-1].copy()
    lat = np.maximum.accumulate(lat, axis=0)
    lat = np.minimum.accumulate(lat, axis=1)
    lat = np.minimum.accumulate(lat, axis=2)
    t = PerfTable("f", [1, 2, 4, 8, 16, 32], list(range(10, 101, 10)), list(range(10, 101, 10)),
                  np.ascontiguousarray(lat))
    n = 100_000
    c = np.column_stack([rng.integers(1, 33, n).astype(float), rng.integers(1, 101, n).astype(float),
                         rng.integers(1, 101, n).astype(float)])
    dc = torch.from_numpy(c).cuda()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    rps = torch.empty_like(out)
    t.predict_latency_many(dc, out, rps)
    want = or_interp3_many(t._b_axis, t._s_axis, t._q_axis, t.latency_ms, c)
    assert same_bits(out.cpu().numpy(), want)
    want_rps = np.array([or_throughput(bb, ll) for bb, ll in zip(c[:2000, 0], want[:2000])])
    assert same_bits(rps.cpu().numpy()[:2000], want_rps)
    # scalar API + error convention (hs/perf.py:88-91)
    assert t.predict_latency(8, 50, 50) == want_at(t, 8, 50, 50)
    assert t.throughput(8, 100, 100) == or_throughput(8, t.latency_ms[3, 9, 9])
    with pytest.raises(ValueError, match="batch"):
        t.predict_latency(33, 50, 50)


def want_at(t, b, s, q):
    return or_interp3_many(t._b_axis, t._s_axis, t._q_axis, t.latency_ms,
                           np.array([[b, s, q]], dtype=float))[0]


def test_throughput_definition():
    from paper_2505_01968_b200 import PerfTable
    t = PerfTable("fn", [8], [100], [100], np.full((1, 1, 1), 20.0))
    assert t.throughput(8, 100, 100) == 400.0
    t1 = PerfTable("fn", [1], [100], [100], np.full((1, 1, 1), 1000.0))
    assert t1.throughput(1, 100, 100) == 1.0


def test_non_strict_axes_use_literal_search(kern):
    """Duplicate axis values (accepted by the reference's raw kernel) follow the literal
    binary search, so even its tie behaviour matches (_grid_cy.pyx:20-26)."""
    b = np.array([1.0, 2.0, 2.0, 2.0, 3.0])
    s = np.array([10.0, 10.0, 20.0])
    q = np.array([5.0, 7.0, 7.0, 9.0])
    rng = np.random.default_rng(1)
    v = np.ascontiguousarray(rng.uniform(1, 9, (5, 3, 4)))
    c = np.column_stack([rng.choice([0.5, 1, 1.5, 2, 2.5, 3, 4], 5000),
                         rng.choice([5, 10, 15, 20, 25], 5000),
                         rng.choice([4, 5, 6, 7, 8, 9, 10], 5000)]).astype(float)
    out = np.empty(len(c))
    kern.interp3_many(b, s, q, v, c, out)
    assert same_bits(out, or_interp3_many(b, s, q, v, c))


def test_literal_kernel_also_bit_exact(interp_golden, tmp_path):
    """RAPP_FORCE_LITERAL=1 routes every table through the literal-search kernel; it must
    reproduce the same golden vectors as the fast path."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r)\n"
        "from tests.conftest import load_golden, golden_table_arrays, fromhex, same_bits\n"
        "from paper_2505_01968_b200 import kernels\n"
        "g = load_golden('interp.json')\n"
        "for rec in g['tables']:\n"
        "    b, s, q, v = golden_table_arrays(rec['table'])\n"
        "    c = fromhex(rec['coords']).reshape(-1, 3); out = np.empty(len(c))\n"
        "    kernels.interp3_many(b, s, q, v, c, out)\n"
        "    assert same_bits(out, fromhex(rec['latency']))\n"
        "print('literal ok')\n") % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RAPP_FORCE_LITERAL="1")
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert res.returncode == 0 and "literal ok" in res.stdout, res.stderr[-2000:]


AXIS_KINDS = {
    "unit": lambda n: np.arange(1.0, n + 1.0),                 # uniform, pow2 step
    "half": lambda n: 0.5 * np.arange(n) - 3.0,                # uniform, step 0.5
    "tens": lambda n: 10.0 * np.arange(1, n + 1),              # uniform step 10 (not pow2)
    "pow2": lambda n: 2.0 ** np.arange(n),                     # geometric (1,2,4,...)
    "tenth": lambda n: 0.1 + np.arange(n),                     # step 1 but inexact nodes
    "irregular": lambda n: np.cumsum(np.random.default_rng(n).uniform(1e-3, 7, n)),
    "tiny": lambda n: 1e-300 * np.arange(1, n + 1),
}


@pytest.mark.parametrize("kind", sorted(AXIS_KINDS))
@pytest.mark.parametrize("n", [1, 2, 3, 17, 100])
def test_axis_layouts_bit_exact(kern, kind, n):
    """Every locate mode of the fast path (uniform arithmetic, exact buckets, corrected
    buckets, pow2 reciprocal vs division) against the oracle, incl. nodes and midpoints."""
    ax = AXIS_KINDS[kind](n).astype(np.float64)
    rng = np.random.default_rng(n * 31 + len(kind))
    b = np.array([1.0, 2.0, 4.0])
    v = np.ascontiguousarray(rng.uniform(1, 100, (3, n, n)))
    m = 60_000
    lo, hi = ax[0], ax[-1]
    span = (hi - lo) if hi > lo else 1.0
    xs = np.concatenate([rng.uniform(lo - 0.1 * span, hi + 0.1 * span, m - 3 * n), ax,
                         (ax[:-1] + ax[1:]) / 2 if n > 1 else ax, np.nextafter(ax, np.inf)])
    xs = xs[:m]
    c = np.column_stack([rng.uniform(0, 5, len(xs)), rng.permutation(xs), xs])
    out = np.empty(len(c))
    kern.interp3_many(b, ax, ax, v, c, out)
    assert same_bits(out, or_interp3_many(b, ax, ax, v, c))


def test_non_positive_and_non_finite_values(kern):
    """Raw-kernel tables with zero, negative, inf or NaN values (the reference kernel
    accepts any doubles) stay bit-exact: they bypass the positive-table fast path."""
    rng = np.random.default_rng(9)
    b = np.array([1.0, 2.0, 4.0, 8.0])
    s = np.arange(1.0, 11.0)
    q = np.arange(10.0, 101.0, 10.0)
    for fill in (0.0, -0.0, -3.5, np.inf, -np.inf, np.nan):
        v = np.ascontiguousarray(rng.uniform(-5, 5, (4, 10, 10)))
        v.flat[rng.integers(0, v.size, 30)] = fill
        c = np.column_stack([rng.uniform(0, 9, 20000), rng.uniform(0, 11, 20000),
                             rng.uniform(0, 110, 20000)])
        c[::7] = np.round(c[::7])
        out = np.empty(len(c))
        kern.interp3_many(b, s, q, v, c, out)
        assert same_bits(out, or_interp3_many(b, s, q, v, c)), fill


@pytest.mark.parametrize("b_axis", [[1, 2, 4, 8, 16, 32], [0.5, 1, 2], [2, 4, 8, 16], [1, 2],
                                    [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024],
                                    [1, 2, 4, 9], [0.25, 0.5, 1.0, 2.0, 4.0]])
def test_batch_axis_modes_bit_exact(kern, b_axis):
    """Geometric power-of-two batch axes (exponent-bit locate) and near-misses (LUT)."""
    b = np.asarray(b_axis, dtype=np.float64)
    s = np.arange(1.0, 101.0)
    q = np.arange(1.0, 101.0)
    rng = np.random.default_rng(len(b_axis))
    v = np.ascontiguousarray(rng.uniform(1, 100, (len(b), 100, 100)))
    m = 100_000
    xb = np.concatenate([rng.uniform(b[0] / 4, b[-1] * 2, m - 3 * len(b)), b,
                         np.nextafter(b, 0), np.nextafter(b, np.inf)])
    c = np.column_stack([xb, rng.uniform(0, 101, m), rng.uniform(0, 101, m)])
    out = np.empty(m)
    kern.interp3_many(b, s, q, v, c, out)
    assert same_bits(out, or_interp3_many(b, s, q, v, c))


def test_config2_stream_large_vs_oracle():
    """Long streams exercise every stage reuse of the TMA ring (a cross-proxy race there
    would show up as rare wrong rows): 12M queries on two config-2 tables, 0 ulp."""
    import torch
    import bench
    from paper_2505_01968_b200 import PerfTable
    dev = torch.device("cuda", 0)
    for mi, (name, b, s, q, v) in list(enumerate(bench.config2_arrays()))[::2]:
        t = PerfTable(name, bench.BATCHES, list(range(1, 101)), list(range(1, 101)), v)
        c = bench.gen_queries(b, s, q, 6_000_000, 77 + mi, dev)
        got = t.predict_latency_many(c).cpu().numpy()
        assert same_bits(got, or_interp3_many(b, s, q, v, c.cpu().numpy())), name


def test_stateless_table_cache_alternating_tables(kern):
    """The stateless entry points keep the last 8 distinct tables resident (exact content
    match): 12 tables of different shapes, called in an interleaved order with evictions,
    in-place segment reuse and tables that differ in one value only, stay bit-exact."""
    rng = np.random.default_rng(21)
    tables = []
    for i in range(12):
        nb, ns, nq = (3 + i % 4, 5 + (i * 7) % 11, 4 + (i * 5) % 9)
        b = np.cumsum(rng.uniform(0.5, 3.0, nb))
        s = np.cumsum(rng.uniform(1.0, 9.0, ns))
        q = np.cumsum(rng.uniform(1.0, 9.0, nq))
        v = rng.uniform(1.0, 100.0, (nb, ns, nq))
        tables.append((b, s, q, v))
    b0, s0, q0, v0 = tables[0]
    v1 = v0.copy()
    v1[1, 2, 3] = np.nextafter(v1[1, 2, 3], np.inf)  # one ulp apart: a different table
    tables.append((b0, s0, q0, v1))
    order = [0, 1, 2, 3, 0, 12, 4, 5, 6, 7, 8, 9, 0, 10, 11, 12, 3, 1, 0, 12]
    for k in order:
        b, s, q, v = tables[k]
        c = np.column_stack([rng.uniform(b[0] - 1, b[-1] + 1, 3000),
                             rng.uniform(s[0] - 1, s[-1] + 1, 3000),
                             rng.uniform(q[0] - 1, q[-1] + 1, 3000)])
        out = np.empty(len(c))
        kern.interp3_many(b, s, q, v, c, out)
        assert same_bits(out, or_interp3_many(b, s, q, v, c)), k


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 63, 511, 513, 9_473, 1_000_003])
@pytest.mark.parametrize("offset", [0, 1])
def test_stream_tails_and_unaligned_coords(n, offset):
    """K2's direct-load walk (32-row slices, grid-stride, next slice prefetched): ragged
    tails, odd lane pairs, 8-byte-misaligned coordinate rows and a guarded output — 0 ulp
    vs the oracle and not one byte written outside the n outputs."""
    import torch
    import bench
    from paper_2505_01968_b200 import PerfTable
    dev = torch.device("cuda", 0)
    name, b, s, q, v = bench.config2_arrays()[1]
    t = PerfTable(name, bench.BATCHES, list(range(1, 101)), list(range(1, 101)), v)
    c = bench.gen_queries(b, s, q, n + 1, 900 + n, dev)
    flat = c.view(-1)[offset:offset + 3 * n]
    coords = flat.view(n, 3)
    guard = torch.full((n + 64,), -7.25, dtype=torch.float64, device=dev)
    out = guard[32:32 + n]
    t.predict_latency_many(coords, out)
    torch.cuda.synchronize()
    g = guard.cpu().numpy()
    assert (g[:32] == -7.25).all() and (g[32 + n:] == -7.25).all()
    assert same_bits(g[32:32 + n], or_interp3_many(b, s, q, v, coords.cpu().numpy()))
