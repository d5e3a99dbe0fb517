"""Run-metrics finalize (hs/sim.py:586-621): the CPU oracle and the device kernel against
the reference's own _finalize outputs captured from real simulations
(tests/golden/metrics.json, gen_golden.py:gen_metrics), plus large random engine states."""

import math
import types

import numpy as np
import pytest

from oracle import metrics_oracle as mo

from .conftest import load_golden


@pytest.fixture(scope="module")
def golden():
    return load_golden("metrics.json")


def fx(h):
    return float.fromhex(h)


def unpack(rec):
    base = {f: fx(b) for f, b in rec["functions"].items()}
    counts = {f: tuple(c) for f, c in rec["counts"].items()}
    lat = {f: [fx(x) for x in v] for f, v in rec["latencies"].items()}
    ivs = [(f, sm, q, fx(s), fx(e)) for f, sm, q, s, e in rec["intervals"]]
    return base, counts, lat, ivs, fx(rec["price"]), fx(rec["sim_end"])


def same(a, b):
    return (math.isnan(a) and math.isnan(b)) or float(a).hex() == float(b).hex()


def check(out, want):
    curve, pcts, cost, cpk = out
    for f, row in want["violation_curve"].items():
        assert [x.hex() for x in curve[f]] == row, f
    for f, d in want["percentiles"].items():
        for k, h in d.items():
            assert same(pcts[f][k], fx(h)), (f, k)
    for f, h in want["cost"].items():
        assert same(cost[f], fx(h)), f
    for f, h in want["cost_per_1k"].items():
        assert same(cpk[f], fx(h)), f


def test_oracle_matches_reference(golden):
    for rec in golden:
        check(mo.finalize(*unpack(rec)), rec["out"])
        check(mo.finalize_np(*unpack(rec)), rec["out"])


def engine_of(base, counts, lat, ivs, price, sim_end):
    eng = types.SimpleNamespace()
    eng.functions = {f: types.SimpleNamespace(baseline_latency_ms=b) for f, b in base.items()}
    eng._counts = {f: types.SimpleNamespace(arrived=c[0], completed=c[1], rejected=c[2])
                   for f, c in counts.items()}
    eng._latencies = lat
    eng._intervals = [types.SimpleNamespace(function_id=f, sm_percent=sm, quota_percent=q,
                                            start_ms=s, end_ms=e) for f, sm, q, s, e in ivs]
    eng.cfg = types.SimpleNamespace(price_per_gpu_hour=price)
    eng._timeline = []
    return eng


@pytest.mark.gpu
def test_device_finalize_matches_reference(golden):
    from paper_2505_01968_b200 import metrics
    for rec in golden:
        args = unpack(rec)
        m = metrics.finalize(engine_of(*args), args[-1])
        check((m.violation_curve, m.percentiles, m.cost, m.cost_per_1k), rec["out"])
        assert m.multipliers == mo.SLO_MULTIPLIERS


@pytest.mark.gpu
def test_device_finalize_large_random_against_oracle():
    """100 functions, up to 200k latencies each (many exact ties, values on the SLO
    thresholds), shuffled intervals — bit-exact against the oracle."""
    from paper_2505_01968_b200 import metrics
    rng = np.random.default_rng(11)
    base, counts, lat, ivs = {}, {}, {}, []
    for i in range(100):
        f = f"fn-{i:03d}"
        b = float(rng.choice([20.0, 12.5, 33.3]))
        n = int(rng.choice([0, 1, 1000, 200_000]))
        vals = np.where(rng.random(n) < 0.2,
                        b * rng.choice(mo.SLO_MULTIPLIERS, n),
                        np.round(rng.uniform(0, 12 * b, n), 2))
        base[f] = b
        lat[f] = vals.tolist()
        rej = int(rng.integers(0, 50))
        counts[f] = (n + rej + int(rng.integers(0, 9)), n, rej)
        for _ in range(int(rng.integers(0, 30))):
            s = float(rng.uniform(0, 1e5))
            e = -1.0 if rng.random() < 0.2 else s + float(rng.uniform(0, 1e5))
            ivs.append((f, int(rng.integers(1, 101)), int(rng.integers(1, 101)), s, e))
    rng.shuffle(ivs)
    args = (base, counts, lat, ivs, 2.48, 250000.0)
    want_curve, want_p, want_c, want_k = mo.finalize_np(*args)
    m = metrics.finalize(engine_of(*args), 250000.0)
    for f in base:
        assert [x.hex() for x in m.violation_curve[f]] == [x.hex() for x in want_curve[f]]
        for k in want_p[f]:
            assert same(m.percentiles[f][k], want_p[f][k]), (f, k)
        assert same(m.cost[f], want_c[f]) and same(m.cost_per_1k[f], want_k[f])
