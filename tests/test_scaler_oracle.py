"""The scaler oracle (oracle/scaler_oracle.py) reproduces the real reference's decisions:
every single-function case and every multi-function tick in the golden vectors (CPU)."""

import copy

import numpy as np
import pytest

from oracle import scaler_oracle as so

from .conftest import golden_table_arrays, load_golden
from .golden_io import (cluster_from, cluster_to, function_from, fx, golden_cluster_to,
                        make_part, make_pod, surface_tables)


class _T:
    """PerfTable-shaped view over golden arrays for the oracle."""

    def __init__(self, rec):
        b, s, q, v = golden_table_arrays(rec)
        self.function_id = rec["function_id"]
        self.batches, self.sms = list(rec["batches"]), list(rec["sms"])
        self._b_axis, self._s_axis, self._q_axis, self.latency_ms = b, s, q, v


def _cfg(c):
    a, b, d, cd, rmin = c
    return {"alpha": fx(a), "beta": fx(b), "delta": d, "cooldown_ms": fx(cd), "r_min": fx(rmin)}


@pytest.fixture(scope="module")
def scale_golden():
    return load_golden("scale.json")


@pytest.fixture(scope="module")
def tick_golden():
    return load_golden("tick.json")


def test_oracle_reproduces_reference_scale_decisions(scale_golden):
    table = so.OTable(_T(scale_golden["table"]))
    fn = function_from(scale_golden["function"])
    assert len(scale_golden["cases"]) > 1500
    for case in scale_golden["cases"]:
        cluster = cluster_from(case["cluster"])
        acts, stamp = so.scale(_cfg(case["cfg"]), fn, table, cluster, fx(case["rate"]),
                               fx(case["last_down"]), make_pod, make_part)
        assert [list(a) for a in acts] == case["actions"], case["name"]
        want_stamp = fx(case["stamp"])
        if case["last_down"] is None:
            assert stamp == want_stamp, case["name"]
        elif stamp is not None:
            assert stamp == want_stamp, case["name"]
        # scale() must not mutate the caller's cluster (it stages on a scratch copy)
        assert cluster_to(cluster) == golden_cluster_to(case["cluster"]), case["name"]


def run_oracle_ticks(run):
    fns = [function_from(f) for f in run["functions"]]
    tables = {k: so.OTable(t) for k, t in surface_tables(run["tables"], fns).items()}
    cluster = cluster_from(run["initial"])
    cfg = {"alpha": fx(run["alpha"]), "beta": fx(run["beta"]), "delta": run["delta"],
           "cooldown_ms": fx(run["cooldown_ms"]), "r_min": fx(run["r_min"])}
    kal = {k: fx(v) for k, v in run["kalman"].items()}
    p0 = kal.pop("P0")
    kstate, last_down = {}, {}
    counter = run["pod_counter0"]
    functions = {f.function_id: f for f in fns}
    per_tick = []
    for t in run["ticks"]:
        arrivals = {f.function_id: a for f, a in zip(fns, t["arrivals"])}
        acts, obs, pred, counter = so.tick(cfg, functions, tables, cluster, fx(t["now"]),
                                           fx(run["interval_ms"]), arrivals, set(t["idle"]),
                                           kstate, kal, p0, last_down, counter, make_pod,
                                           make_part, cold_start_ms=fx(run["cold_start_ms"]),
                                           policy=run.get("policy", "hybrid"))
        per_tick.append((acts, obs, pred))
    return per_tick, cluster


def test_oracle_reproduces_reference_ticks(tick_golden):
    for run in tick_golden["runs"]:
        per_tick, cluster = run_oracle_ticks(run)
        fids = [f["id"] for f in run["functions"]]
        for t, (acts, obs, pred) in zip(run["ticks"], per_tick):
            want = [list(a) for a in t["actions"]]
            # the reference emits horizontal_up with pod_id None; the oracle reports the
            # id the tick assigned on apply, in order
            new_ids = iter(t["new_pods"])
            for a in want:
                if a[1] == "horizontal_up":
                    a[5] = next(new_ids)
            assert [list(a) for a in acts] == want
            assert [obs[f] for f in fids] == [fx(x) for x in t["observed"]]
            assert [pred[f] for f in fids] == [fx(x) for x in t["predicted"]]
        assert cluster_to(cluster) == golden_cluster_to(run["final"])


def test_oracle_reproduces_reference_replica_policies():
    """hs/policies.py:69-141 (horizontal-only, exclusive-gpu) on randomized clusters."""
    g = load_golden("policy.json")
    table = so.OTable(_T(g["table"]))
    from paper_2505_01968_b200.core import FunctionSpec, PodConfig
    for case in g["cases"]:
        init = case["initial"]
        fn = FunctionSpec("conf-fn", 20.0, perf_table_ref="conf-fn", allowed_batches=[8],
                          initial=PodConfig(*init))
        shape = (init[0], 100, 100) if case["policy"] == "exclusive-gpu" else tuple(init)
        cluster = cluster_from(case["cluster"])
        acts, stamp = so.replica_decide(_cfg(case["cfg"]), fn, table, cluster,
                                        fx(case["rate"]), fx(case["last_down"]), shape,
                                        make_pod, make_part)
        assert [list(a) for a in acts] == case["actions"]
        if stamp is not None:
            assert stamp == fx(case["stamp"])
