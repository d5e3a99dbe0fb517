"""K3 fused lattice search vs the reference's golden most_efficient_config results and the
oracle (exact (b, s, q)).  Mirrors pkg/tests/test_perf.py:170-207 and acceptance C5."""

import os
import random

import numpy as np
import pytest

from oracle.binding import or_most_efficient_config

from .conftest import golden_table_arrays

pytestmark = pytest.mark.gpu


def _table(rec):
    from paper_2505_01968_b200 import PerfTable
    b, s, q, v = golden_table_arrays(rec)
    return PerfTable(rec["function_id"], rec["batches"], rec["sms"], rec["quotas"], v)


def test_golden_search_cases(mec_golden):
    tables = {t["function_id"]: _table(t) for t in mec_golden["tables"]}
    for case in mec_golden["cases"]:
        t = tables[case["table"]]
        got = t.most_efficient_config(float.fromhex(case["target"]), quota_step=case["step"],
                                      batches=case["batches"])
        assert list(got) == case["result"], case


def test_golden_cases_batched_in_one_pass(mec_golden):
    from paper_2505_01968_b200 import PerfTableSet
    tables = {t["function_id"]: _table(t) for t in mec_golden["tables"]}
    by_step = {}
    for case in mec_golden["cases"]:
        by_step.setdefault(case["step"], []).append(case)
    for step, cases in by_step.items():
        ts = PerfTableSet([(tables[c["table"]], c["batches"]) for c in cases], quota_step=step)
        got = ts.search([float.fromhex(c["target"]) for c in cases])
        assert [list(g) for g in got] == [c["result"] for c in cases]


def test_bad_inputs_raise_value_error(mec_golden):
    t = _table(mec_golden["tables"][0])
    with pytest.raises(ValueError):
        t.most_efficient_config(0.0)
    with pytest.raises(ValueError):
        t.most_efficient_config(1.0, quota_step=0)


def _synth(rng, nb, ns, nq, fid):
    """Separable surface of pkg/scripts/gen_tables.py:26-29 with random parameters."""
    from paper_2505_01968_b200 import PerfTable
    bs = sorted(rng.sample(range(1, 33), nb))
    ss = sorted(rng.sample(range(1, 101), ns))
    qs = sorted(rng.sample(range(1, 101), nq))
    fixed, per, floor = rng.uniform(4, 20), rng.uniform(0.5, 4), rng.uniform(0.2, 0.4)
    lat = np.array([[[(fixed + per * b) * (floor + (1 - floor) * (100.0 / s)) * (100.0 / q)
                      for q in qs] for s in ss] for b in bs])
    return PerfTable(fid, bs, ss, qs, lat)


def test_random_tables_targets_steps_vs_oracle():
    from paper_2505_01968_b200 import PerfTableSet
    rng = random.Random(99)
    fns, targets, steps = [], [], []
    for i in range(60):
        t = _synth(rng, rng.randint(1, 6), rng.randint(1, 12), rng.randint(1, 12), f"f{i}")
        allowed = rng.choice([None, list(range(1, 33)), [3, 5, 7], [t.batches[-1]], [1000]])
        peak = t.throughput(t.batches[-1], t.sms[-1], 100)
        frac = rng.choice([0.01, 0.3, 0.5, 0.9, 1.0, 1.5])
        fns.append((t, allowed))
        targets.append(frac * peak)
    for step in (1, 3, 10, 33):
        ts = PerfTableSet(fns, quota_step=step)
        got = ts.search(targets)
        for (t, allowed), target, g in zip(fns, targets, got):
            want = or_most_efficient_config(t._b_axis, t._s_axis, t._q_axis, t.latency_ms,
                                            target, step, allowed)
            assert g == want, (t.function_id, target, step, allowed)


def test_tie_targets_equal_to_lattice_throughput():
    """Targets exactly equal to a lattice point's rps (the `>=` edge, hs/perf.py:132)."""
    from oracle.binding import or_interp3_many, or_throughput
    from paper_2505_01968_b200 import PerfTableSet
    rng = random.Random(5)
    t = _synth(rng, 6, 10, 10, "tie")
    fns, targets = [], []
    for _ in range(200):
        b = rng.randint(1, 32)
        s = rng.choice(t.sms)
        q = rng.randint(1, 100)
        if not (t.batches[0] <= b <= t.batches[-1]):
            continue
        lat = or_interp3_many(t._b_axis, t._s_axis, t._q_axis, t.latency_ms,
                              np.array([[b, s, q]], dtype=float))[0]
        fns.append((t, list(range(1, 33))))
        targets.append(or_throughput(b, lat))
    ts = PerfTableSet(fns, quota_step=1)
    for target, g in zip(targets, ts.search(targets)):
        assert g == or_most_efficient_config(t._b_axis, t._s_axis, t._q_axis, t.latency_ms,
                                             target, 1, list(range(1, 33)))


def test_config5_shaped_functions_vs_oracle():
    """A slice of the 10^9-point config-5 workload: 32 x 100 x 100 lattice per function."""
    from paper_2505_01968_b200 import PerfTableSet
    import bench
    tables = bench.make_config5_tables(8, seed=0)
    allowed = list(range(1, 33))
    ts = PerfTableSet([(t, allowed) for t in tables], quota_step=1)
    assert ts.points == 8 * 32 * 100 * 100
    targets = [0.5 * bench.max_lattice_rps(t) for t in tables]
    got = ts.search(targets)
    for t, target, g in zip(tables[:3], targets[:3], got[:3]):
        assert g == or_most_efficient_config(t._b_axis, t._s_axis, t._q_axis, t.latency_ms,
                                             target, 1, allowed)


def test_config5_full_size_every_function_and_repeatable():
    """BASELINE config 5 at full size: 3,125 functions x 32 x 100 x 100 = 10^9 lattice
    points in one pass.  Two runs give identical decisions (order-independent packed-key
    reduction), and EVERY function's (b, s, q) equals the C oracle (hs/perf.py:104-145),
    which walks all 10^9 points on the host cores (ctypes releases the GIL: one thread per
    core)."""
    import concurrent.futures
    import bench
    from paper_2505_01968_b200 import PerfTableSet
    tables = bench.make_config5_tables(3125, seed=0, device=0)
    allowed = list(range(1, 33))
    ts = PerfTableSet([(t, allowed) for t in tables], quota_step=1)
    assert ts.points == 3125 * 32 * 100 * 100
    rng = np.random.default_rng(17)
    scale = rng.choice([0.001, 0.3, 0.5, 0.9, 1.5], 3125)  # 1.5 x max: the fallback branch
    targets = [float(s * bench.max_lattice_rps(t)) for s, t in zip(scale, tables)]
    first = ts.search(targets)
    assert ts.search(targets) == first

    def oracle(f):
        t = tables[f]
        return or_most_efficient_config(t._b_axis, t._s_axis, t._q_axis, t.latency_ms,
                                        targets[f], 1, allowed)
    with concurrent.futures.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as pool:
        want = list(pool.map(oracle, range(3125)))
    bad = [f for f in range(3125) if first[f] != want[f]]
    assert not bad, (len(bad), bad[:5])


def _rough(rng, nb, ns, nq, fid):
    """Random monotone grid (positive; latency non-decreasing in batch, non-increasing in sm
    and quota, as the loader requires) whose batch growth is superlinear in places, so
    feasibility is not monotone in b."""
    from paper_2505_01968_b200 import PerfTable
    bs = sorted(rng.sample(range(1, 33), nb))
    ss = sorted(rng.sample(range(1, 101), ns))
    qs = sorted(rng.sample(range(1, 101), nq))
    gb = np.cumsum([rng.uniform(0.5, 8.0) * (rng.random() < 0.5 and 6.0 or 1.0)
                    for _ in bs])
    gs = np.cumsum([rng.uniform(0.1, 1.0) for _ in ss])[::-1]
    gq = np.cumsum([rng.uniform(0.1, 1.0) for _ in qs])[::-1]
    lat = gb[:, None, None] * gs[None, :, None] * gq[None, None, :] + rng.uniform(0.1, 2.0)
    return PerfTable(fid, bs, ss, qs, lat)


def test_sparse_batch_lists_and_rough_tables_vs_oracle():
    """K3's run formulation: batch lists that skip table rows, hit only nodes, start or end
    on the axis ends, single-row tables; pair counts that leave ragged per-thread tails."""
    from paper_2505_01968_b200 import PerfTableSet
    rng = random.Random(2024)
    fns, targets = [], []
    for i in range(80):
        t = _rough(rng, rng.randint(1, 7), rng.randint(1, 37), rng.randint(1, 23), f"r{i}")
        lo, hi = t.batches[0], t.batches[-1]
        allowed = rng.choice([
            None, [lo, hi], [hi], [lo], list(t.batches), sorted(rng.sample(range(1, 33), 5)),
            list(range(lo, hi + 1, 3)), [b for b in range(1, 33) if b not in t.batches]])
        if allowed is not None and not any(lo <= b <= hi for b in allowed):
            allowed = None
        peak = max(t.throughput(b, t.sms[-1], 100) for b in t.batches)
        fns.append((t, allowed))
        targets.append(rng.choice([0.05, 0.4, 0.7, 0.95, 1.0, 2.0]) * peak)
    for step in (1, 7, 25):
        ts = PerfTableSet(fns, quota_step=step)
        got = ts.search(targets)
        for (t, allowed), target, g in zip(fns, targets, got):
            want = or_most_efficient_config(t._b_axis, t._s_axis, t._q_axis, t.latency_ms,
                                            target, step, allowed)
            assert g == want, (t.function_id, target, step, allowed)
