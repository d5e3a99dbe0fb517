#!/usr/bin/env python3
"""Generates the golden vectors in tests/golden/ by running the REAL reference.

Run in the build container only (the reference tree is absent on the GPU box):

    python tests/golden/gen_golden.py            # all sets
    python tests/golden/gen_golden.py interp mec # selected sets

The reference package is imported from a scratch copy (/tmp/refpkg) whose
Cython kernel is built in place, because /root/reference is read-only.
Doubles are stored as float.hex() strings so comparisons are 0-ulp.
"""

from __future__ import annotations

import json
import os
import random
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
if ROOT not in sys.path:
    sys.path.append(ROOT)  # bench.py (world builders); after the reference's own `tests`
REF_PKG = "/root/reference/pkg"
SCRATCH = "/tmp/refpkg"


def import_reference():
    if not os.path.exists(os.path.join(SCRATCH, "src", "hybridscale")):
        shutil.copytree(REF_PKG, SCRATCH)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                       check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    sys.path.insert(0, SCRATCH)  # for `tests.conftest` / `tests.oracles`
    import hybridscale
    assert hybridscale.KERNEL_BACKEND == "cython", hybridscale.KERNEL_BACKEND
    return hybridscale


def hx(x: float) -> str:
    return float(x).hex()


def hx_arr(a) -> list[str]:
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def table_dict(t) -> dict:
    return {"function_id": t.function_id, "batches": list(t.batches), "sms": list(t.sms),
            "quotas": list(t.quotas), "latency_ms": hx_arr(t.latency_ms)}


def dump(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


# -- interpolation ------------------------------------------------------------


def gen_interp(hs):
    from hybridscale import load_table
    from hybridscale._kernels import _grid_cy, locate
    tables = [load_table(os.path.join(REF_PKG, "tables", n))
              for n in ("resnet50.csv", "bert-small.csv")]
    # the test_kernels.py:_grid() table (pkg/tests/test_kernels.py:12-19)
    from tests.test_kernels import _grid
    b, s, q, v = _grid()
    grid_tab = hs.PerfTable("kernels-grid", [1, 2, 4, 8], [25, 50, 75, 100],
                            [10, 40, 70, 100], v)
    tables.append(grid_tab)
    rng = np.random.default_rng(20261017)
    out = {"tables": [], "locate": []}
    for t in tables:
        n = 3000
        c = np.column_stack([
            rng.uniform(t.batches[0] - 1, t.batches[-1] + 1, n),
            rng.uniform(t.sms[0] - 10, t.sms[-1] + 10, n),
            rng.uniform(t.quotas[0] - 10, t.quotas[-1] + 10, n)])
        # exact node hits, clamps, integers and specials
        c[0::9, 0] = rng.choice(t.batches, len(c[0::9]))
        c[1::9, 1] = rng.choice(t.sms, len(c[1::9]))
        c[2::9, 2] = rng.choice(t.quotas, len(c[2::9]))
        c[3::11] = np.round(c[3::11])
        c[5] = [np.nan, 50.0, 50.0]
        c[6] = [2.0, np.nan, 50.0]
        c[7] = [2.0, 50.0, np.nan]
        c[8] = [np.inf, -np.inf, 1e308]
        c[9] = [-0.0, 0.0, -1e-300]
        res = np.empty(n)
        _grid_cy.interp3_many(t._b_axis, t._s_axis, t._q_axis, t.latency_ms, c, res)
        out["tables"].append({"table": table_dict(t), "coords": hx_arr(c),
                              "latency": hx_arr(res)})
    axis = np.array([10.0, 20.0, 40.0])
    for x in [10.0, 20.0, 40.0, 25.0, 5.0, 99.0, 39.999999, 10.000001, float("nan"),
              float("inf"), float("-inf"), -0.0]:
        lo, hi, t = locate(axis, x)
        out["locate"].append({"axis": hx_arr(axis), "x": hx(x), "lo": lo, "hi": hi,
                              "t": hx(t)})
    one = np.array([7.0])
    for x in [7.0, 1.0, 9.0, float("nan")]:
        lo, hi, t = locate(one, x)
        out["locate"].append({"axis": hx_arr(one), "x": hx(x), "lo": lo, "hi": hi,
                              "t": hx(t)})
    dump("interp.json", out)


# -- most_efficient_config ------------------------------------------------------


def gen_mec(hs):
    from hybridscale import load_table
    from tests.conftest import make_conformance_table, random_monotone_table
    tables = [load_table(os.path.join(REF_PKG, "tables", n))
              for n in ("resnet50.csv", "bert-small.csv")]
    tables.append(make_conformance_table())
    rng = random.Random(4242)
    for i in range(12):
        tables.append(random_monotone_table(rng, rng.randint(1, 5), rng.randint(1, 5),
                                            rng.randint(1, 6), function_id=f"rand-{i}"))
    cases = []
    for t in tables:
        peak = t.throughput(t.batches[-1], t.sms[-1], 100)
        targets = [0.001, 0.1 * peak, 0.3 * peak, 0.5 * peak, 0.75 * peak, 0.99 * peak,
                   peak, 2.0 * peak, 1e9]
        # tie edge: targets exactly equal to a lattice throughput
        for _ in range(4):
            b = rng.choice(t.batches)
            s = rng.choice(t.sms)
            qq = rng.choice(range(10, 101, 10))
            targets.append(t.throughput(b, s, qq))
        for step in (1, 7, 10, 20, 25, 50, 100):
            for batches in (None, t.batches[:1], [3, 5], [0, 1000], [t.batches[-1], 1]):
                for target in targets:
                    got = t.most_efficient_config(target, quota_step=step, batches=batches)
                    cases.append({"table": t.function_id, "target": hx(target),
                                  "step": step, "batches": batches, "result": list(got)})
    dump("mec.json", {"tables": [table_dict(t) for t in tables], "cases": cases})


# -- scaler decisions (Autoscaler.scale) ------------------------------------------------


def cluster_dict(cluster) -> dict:
    return {
        "clock_ms": hx(cluster.clock_ms),
        "gpus": [{"id": g.gpu_id, "partitions": [
            {"sm": p.sm_percent, "residents": list(p.resident_pods), "alloc": p.quota_allocated}
            for p in g.partitions]} for g in cluster.gpus.values()],
        "pods": [{"id": p.pod_id, "fid": p.function_id, "b": p.batch, "s": p.sm_percent,
                  "q": p.quota_percent, "gpu": p.gpu_id, "state": p.state.value}
                 for p in cluster.pods.values()],
    }


def action_list(actions) -> list:
    return [[a.function_id, a.kind.value, a.batch, a.sm_percent, a.quota_percent, a.pod_id,
             a.gpu_id] for a in actions]


def fn_dict(f) -> dict:
    return {"id": f.function_id, "table": f.perf_table_ref or f.function_id,
            "min_rps": None if f.min_rps is None else hx(f.min_rps),
            "allowed": list(f.allowed_batches),
            "initial": [f.initial.batch, f.initial.sm_percent, f.initial.quota_percent,
                        f.initial.replicas]}


def gen_scale(hs):
    """Single-function decisions: the six hand-traced scenarios (test_acceptance.py C2),
    the extra branch cases of test_autoscaler.py and its three randomized loops."""
    import copy
    from hybridscale import Autoscaler, ScalerConfig, build_cluster
    from tests.conftest import make_conformance_table, make_function, place_running_pod
    from tests.test_acceptance import _conformance_scenarios
    from tests.test_autoscaler import _random_cluster

    cfg = ScalerConfig(alpha=0.9, beta=0.5, delta_iq=20, cooldown_ms=30000, r_min=1.0)
    table = make_conformance_table()
    fn = make_function("conf-fn")
    cases = []

    def record(name, cluster, rate, last_down=None, config=cfg):
        sc = Autoscaler(config, {"conf-fn": table})
        if last_down is not None:
            sc._last_scale_down["conf-fn"] = last_down
        before = cluster_dict(cluster)
        acts = sc.scale(fn, copy.deepcopy(cluster), rate)
        cases.append({"name": name, "cluster": before, "rate": hx(rate),
                      "last_down": None if last_down is None else hx(last_down),
                      "cfg": [hx(config.alpha), hx(config.beta), config.delta_iq,
                              hx(config.cooldown_ms), hx(config.r_min)],
                      "actions": action_list(acts),
                      "stamp": None if "conf-fn" not in sc._last_scale_down else
                      hx(sc._last_scale_down["conf-fn"])})

    for name, build, rate, _ in _conformance_scenarios():
        record(name, build(), rate)
    c = build_cluster(2, functions=[make_function("conf-fn")])
    place_running_pod(c, "p0", "conf-fn", 8, 50, 100, "gpu-000")
    place_running_pod(c, "other", "other-fn", 1, 50, 100, "gpu-000")
    record("fresh-gpu fallback", c, 1000.0)
    c = build_cluster(3, functions=[make_function("conf-fn")])
    place_running_pod(c, "pa", "conf-fn", 8, 25, 20, "gpu-000")
    place_running_pod(c, "pb", "conf-fn", 8, 50, 20, "gpu-000")
    record("vertical before horizontal", c, 500.0)
    c = build_cluster(3, functions=[make_function("conf-fn")])
    place_running_pod(c, "p0", "conf-fn", 8, 50, 100, "gpu-000")
    c.clock_ms = 60_000.0
    record("cooldown blocks", c, 50.0, last_down=50_000.0)
    c.clock_ms = 80_001.0
    record("cooldown expired", c, 50.0, last_down=50_000.0)
    for seed, lo, hi, kind in ((99, 0, 600, "legal"), (7, None, None, "cover"),
                               (31, 1.01, 20, "last-pod")):
        rng = random.Random(seed)
        for trial in range(300 if kind != "last-pod" else 200):
            cluster = _random_cluster(rng)
            if kind == "cover":
                pods = cluster.pods_of("conf-fn")
                cap = sum(table.throughput(8, p.sm_percent, p.quota_percent) for p in pods)
                rate = rng.uniform(cap, cap * 3 + 50)
            else:
                rate = rng.uniform(lo, hi)
            for step in (20, 7):
                conf = ScalerConfig(alpha=0.9, beta=0.5, delta_iq=step, cooldown_ms=30000,
                                    r_min=1.0)
                record(f"{kind}-{trial}-d{step}", cluster, rate, config=conf)
    dump("scale.json", {"table": table_dict(table), "function": fn_dict(fn), "cases": cases})


# -- whole scaler ticks (SimulationEngine._handle_scaler) --------------------------------


def make_tick_world(hs, nfn, ngpu, seed, ns=10, nq=10, allowed_all=False):
    """Functions with random gen_tables-style surfaces and a cluster."""
    from hybridscale import FunctionSpec, PerfTable, PodConfig, build_cluster
    rng = random.Random(seed)
    bs = [1, 2, 4, 8, 16, 32]
    ss = list(range(100 // ns, 101, 100 // ns))
    qs = list(range(100 // nq, 101, 100 // nq))
    tables, fns, params = {}, [], []
    for i in range(nfn):
        fid = f"fn-{i:04d}"
        fixed, per, floor = rng.uniform(4, 20), rng.uniform(0.5, 4), rng.uniform(0.2, 0.4)
        params.append([hx(fixed), hx(per), hx(floor)])
        lat = np.array([[[(fixed + per * b) * (floor + (1.0 - floor) * (100.0 / s)) * (100.0 / q)
                          for q in qs] for s in ss] for b in bs])
        tables[fid] = PerfTable(fid, bs, ss, qs, lat)
        allowed = list(range(1, 33)) if allowed_all else rng.choice([[8], [1, 2, 4, 8], [4, 8, 16]])
        fns.append(FunctionSpec(function_id=fid, baseline_latency_ms=20.0, perf_table_ref=fid,
                                min_rps=rng.choice([None, 1.0, 5.0]), allowed_batches=allowed,
                                initial=PodConfig(8, rng.choice([20, 25, 30]), 20, 1)))
    cluster = build_cluster(ngpu, functions=fns)
    return fns, tables, cluster, {"batches": bs, "sms": ss, "quotas": qs, "params": params}


def gen_tick(hs):
    """Multi-tick runs of the reference's per-tick loop.  Arrivals and the set of idle pods
    are drawn per tick; the engine's own bootstrap places the initial pods."""
    from hybridscale import ScalerConfig, SimConfig, WorkloadTrace
    from hybridscale.sim import SimulationEngine
    runs = []
    specs = [  # (nfn, ngpu, seed, ticks, delta, alpha, beta, policy)
        (12, 6, 1, 8, 10, 0.9, 0.5, "hybrid"), (40, 16, 2, 8, 10, 0.65, 0.45, "hybrid"),
        (100, 64, 3, 8, 10, 0.9, 0.5, "hybrid"), (60, 20, 4, 8, 20, 0.8, 0.3, "hybrid"),
        (30, 40, 5, 8, 1, 0.9, 0.5, "hybrid"),
        (20, 12, 6, 8, 10, 0.9, 0.5, "horizontal-only"),
        (50, 30, 7, 8, 10, 0.65, 0.45, "horizontal-only"),
        (10, 24, 8, 8, 10, 0.9, 0.5, "exclusive-gpu"),
        (30, 40, 9, 8, 10, 0.8, 0.3, "exclusive-gpu"),
    ]
    if os.environ.get("GOLDEN_BIG"):
        specs.append((1000, 400, 0, 1, 10, 0.9, 0.5, "hybrid"))
    for nfn, ngpu, seed, nticks, delta, alpha, beta, policy in specs:
        fns, tables, cluster, tparams = make_tick_world(hs, nfn, ngpu, seed)
        cfg = ScalerConfig(alpha=alpha, beta=beta, delta_iq=delta, cooldown_ms=3000.0, r_min=1.0)
        simcfg = SimConfig(scaler_interval_ms=1000.0, cold_start_ms=1500.0)
        trace = WorkloadTrace(entries=[], horizon_ms=1.0) if hasattr(hs, "WorkloadTrace") else None
        kal = {"A": 1.0, "Q": 25.0, "H": 1.0, "D": 4.0, "P0": 1.0}
        eng = SimulationEngine(trace, fns, tables, cluster, cfg, simcfg, policy, kal)
        eng._bootstrap()
        recorded = []
        orig = eng.policy.decide

        def spy(function, cl, rate, _orig=orig):
            acts = _orig(function, cl, rate)
            recorded.extend(acts)
            return acts
        eng.policy.decide = spy
        rng = random.Random(seed * 7919)
        run = {"nfn": nfn, "ngpu": ngpu, "seed": seed, "policy": policy, "delta": delta,
               "alpha": hx(alpha),
               "beta": hx(beta), "cooldown_ms": hx(3000.0), "r_min": hx(1.0),
               "interval_ms": hx(1000.0), "cold_start_ms": hx(1500.0),
               "kalman": {k: hx(v) for k, v in kal.items()},
               "functions": [fn_dict(f) for f in fns],
               "tables": tparams,
               "initial": cluster_dict(eng.cluster), "ticks": []}
        shape_sq = (100, 100) if policy == "exclusive-gpu" else None
        caps = {f.function_id: tables[f.function_id].throughput(
                    8, *(shape_sq or (f.initial.sm_percent, 20))) for f in fns}
        counter0 = eng._pod_counter
        run["pod_counter0"] = counter0
        for k in range(nticks):
            now = 1000.0 * (k + 1)
            # load swings (up, up, collapse, ...) so pods are added and then drained
            swing = (2.5, 3.5, 0.15, 0.05, 2.0, 0.3, 4.0, 0.02)[k % 8]
            arrivals = {f.function_id: int(rng.uniform(0.2, 1.5) * swing * caps[f.function_id])
                        for f in fns}
            busy = {pid for pid in eng._runtimes if rng.random() < 0.3}
            for pid, rt in eng._runtimes.items():
                rt.in_service = [] if pid in busy else None
                rt.queue.clear()
            for fid, a in arrivals.items():
                eng._tick_arrivals[fid] = a
            # ready events at or before `now` precede the scaler tick (hs/sim.py:40-44)
            for pid, rt in list(eng._runtimes.items()):
                if rt.pod.state.value == "cold_starting" and rt.pod.ready_at_ms <= now:
                    eng._handle_ready(now, pid)
            idle = sorted(pid for pid in eng._runtimes if pid not in busy)
            recorded.clear()
            before = cluster_dict(eng.cluster)
            n_before = eng._pod_counter
            eng._handle_scaler(now)
            tl = eng._timeline[-nfn:]
            run["ticks"].append({
                "now": hx(now), "arrivals": [arrivals[f.function_id] for f in fns],
                "idle": idle,
                "actions": action_list(recorded),
                "new_pods": [f"pod-{i:06d}" for i in range(n_before, eng._pod_counter)],
                "observed": [hx(p.observed_rps) for p in tl],
                "predicted": [hx(p.predicted_rps) for p in tl]})
            for rt in eng._runtimes.values():
                rt.in_service = None
        run["final"] = cluster_dict(eng.cluster)
        runs.append(run)
    dump("tick.json", {"runs": runs})


def gen_policy(hs):
    """Replica-count baseline decisions (hs/policies.py:69-141) on the randomized clusters
    of test_autoscaler.py, plus the hand cases of test_policies.py."""
    import copy
    from hybridscale import ScalerConfig, build_cluster, make_policy
    from tests.conftest import make_conformance_table, make_function, place_running_pod
    from tests.test_autoscaler import _random_cluster
    table = make_conformance_table()
    cases = []
    for pname in ("horizontal-only", "exclusive-gpu"):
        for seed, lo, hi in ((11, 0, 600), (12, 1.01, 60), (13, 100, 3000)):
            rng = random.Random(seed)
            for trial in range(150):
                cluster = _random_cluster(rng)
                cluster.clock_ms = rng.choice([0.0, 20_000.0, 60_000.0])
                rate = rng.uniform(lo, hi)
                init = rng.choice([(8, 50, 20), (8, 25, 40), (8, 50, 10)])
                fn = make_function("conf-fn", initial=init)
                for step in (20, 10):
                    conf = ScalerConfig(alpha=0.9, beta=0.5, delta_iq=step, cooldown_ms=30000,
                                        r_min=1.0)
                    pol = make_policy(pname, conf, {"conf-fn": table})
                    last = rng.choice([None, 10_000.0])
                    if last is not None:
                        pol._last_scale_down["conf-fn"] = last
                    before = cluster_dict(cluster)
                    acts = pol.decide(fn, copy.deepcopy(cluster), rate)
                    cases.append({"policy": pname, "cluster": before, "rate": hx(rate),
                                  "initial": list(init), "last_down": None if last is None
                                  else hx(last),
                                  "cfg": [hx(0.9), hx(0.5), step, hx(30000.0), hx(1.0)],
                                  "actions": action_list(acts),
                                  "stamp": None if "conf-fn" not in pol._last_scale_down
                                  else hx(pol._last_scale_down["conf-fn"])})
    dump("policy.json", {"table": table_dict(table), "cases": cases})


# -- table ingest ----------------------------------------------------------------


def ingest_cases():
    """CSV texts covering the reference's ingest paths (hs/perf.py:155-267): valid tables
    (strict form and csv-module form), duplicates, missing cells, non-positive and
    non-monotone cells, NaN, and every format error class."""
    H = "function_id,batch,sm_percent,quota_percent,latency_ms"
    rng = random.Random(4242)
    cases = {}

    def rows_of(fid, bs, ss, qs, f):
        return [(fid, b, s, q, f(b, s, q)) for b in bs for s in ss for q in qs]

    def text(rows, header=H, sep="\n"):
        return sep.join([header] + [",".join(str(x) for x in r) for r in rows]) + sep

    def surf(b, s, q):
        return (8.0 + 1.5 * b) * (0.35 + 0.65 * (100.0 / s)) * (100.0 / q)

    for name in ("resnet50.csv", "bert-small.csv"):
        cases["ref_" + name] = open(os.path.join(REF_PKG, "tables", name), encoding="utf-8").read()
    base = rows_of("fn", [1, 2, 4, 8], [20, 50, 100], [10, 40, 70, 100], surf)
    cases["valid"] = text(base)
    shuffled = list(base)
    rng.shuffle(shuffled)
    cases["valid_shuffled"] = text(shuffled)
    cases["valid_crlf"] = text(base, sep="\r\n")
    cases["valid_padded"] = text([(" fn ", b, f" {s}", q, f" {v!r}") for fn, b, s, q, v in base])
    cases["valid_quoted"] = H + "\n" + "".join(f'"fn",{b},{s},{q},"{v!r}"\n'
                                                for _, b, s, q, v in base)
    cases["valid_blank_lines"] = text(base[:5]) + "\n\n" + text(base[5:], header="")[1:]
    cases["valid_float_forms"] = text([(fn, b, s, q, f"{v:.6e}" if i % 3 == 0 else
                                        (f"+{v}" if i % 3 == 1 else repr(v)))
                                       for i, (fn, b, s, q, v) in enumerate(base)])
    cases["valid_no_trailing_newline"] = text(base)[:-1]
    cases["valid_single_cell"] = text([("one", 4, 50, 50, 12.5)])
    cases["valid_flat"] = text(rows_of("flat", [1, 2], [50, 100], [50, 100],
                                       lambda b, s, q: 10.0))
    cases["duplicate"] = text(base + [base[3], base[0], base[3]])
    cases["duplicate_shuffled"] = text(shuffled[:20] + [shuffled[2]] + shuffled[20:] +
                                       [shuffled[7]])
    missing = list(base)
    del missing[13]
    del missing[-1]
    cases["missing"] = text(missing)
    cases["missing_and_bad"] = text([(fn, b, s, q, -v if i == 3 else v)
                                     for i, (fn, b, s, q, v) in enumerate(missing)])
    cases["non_positive"] = text([(fn, b, s, q, 0.0 if i == 5 else (-1.5 if i == 30 else v))
                                  for i, (fn, b, s, q, v) in enumerate(base)])
    cases["mono_batch"] = text([(fn, b, s, q, v / 10 if b == 4 else v) for fn, b, s, q, v in base])
    cases["mono_sm"] = text([(fn, b, s, q, v * 3 if s == 100 and q == 40 else v)
                             for fn, b, s, q, v in base])
    cases["mono_quota"] = text([(fn, b, s, q, v * 9 if q == 70 else v) for fn, b, s, q, v in base])
    cases["nan_and_inf"] = text([(fn, b, s, q, "nan" if i == 7 else ("inf" if i == 9 else v))
                                 for i, (fn, b, s, q, v) in enumerate(base)])
    cases["many_issues"] = text([(fn, b, s, q, (-v if i % 7 == 0 else v * (1 + (i % 5))))
                                 for i, (fn, b, s, q, v) in enumerate(base)])
    cases["bad_header"] = "nope,nope\n1,2\n"
    cases["header_only"] = H + "\n"
    cases["empty_file"] = ""
    cases["mixed_ids"] = text(base[:10] + [("other",) + tuple(base[10][1:])] + base[11:])
    cases["bad_int"] = text(base[:4] + [("fn", "x", 20, 10, 1.0)] + base[4:])
    cases["bad_float"] = text(base[:4] + [("fn", 1, 20, 10, "fast")] + base[4:])
    cases["short_row"] = H + "\n" + "fn,1,20\n" + text(base, header="")[1:]
    cases["float_int_field"] = text(base[:2] + [("fn", "1.0", 20, 10, 1.0)] + base[2:])
    cases["underscore_int"] = text([(fn, b, "1_00" if s == 100 else s, q, v)
                                    for fn, b, s, q, v in base])
    cases["negative_axes"] = text(rows_of("neg", [-4, 2], [-50, 100], [10, 20],
                                          lambda b, s, q: 100.0 - b - s / 10.0 - q))
    cases["big_batch_values"] = text(rows_of("big", [1, 10 ** 12], [50, 100], [10, 100],
                                             lambda b, s, q: 5.0 + (b > 1) - s / 100.0 - q / 1000.0))
    return cases


def gen_ingest(hs):
    import tempfile
    from hybridscale import load_table, validate_table_file
    from hybridscale.errors import TableFormatError
    out = {}
    tmp = tempfile.mkdtemp()
    for name, body in ingest_cases().items():
        path = os.path.join(tmp, "table.csv")
        with open(path, "w", encoding="utf-8", newline="") as fh:
            fh.write(body)
        rep = validate_table_file(path)
        rec = {"csv": body, "report": {
            "function_id": rep.function_id, "batches": list(rep.batches), "sms": list(rep.sms),
            "quotas": list(rep.quotas),
            "issues": [[i.kind, i.message, list(i.coord) if i.coord else None]
                       for i in rep.issues]}}
        try:
            t = load_table(path)
            rec["load"] = {"ok": True, "table": table_dict(t)}
        except TableFormatError as exc:
            msg = str(exc)
            assert msg.startswith(path + ": "), msg
            rec["load"] = {"ok": False, "message": msg[len(path) + 2:]}
        out[name] = rec
    dump("ingest.json", out)


# -- run metrics finalize --------------------------------------------------------------


def _finalize_record(eng, sim_end, out):
    def ivd(iv):
        return [iv.function_id, iv.sm_percent, iv.quota_percent, hx(iv.start_ms), hx(iv.end_ms)]
    return {
        "functions": {f: hx(eng.functions[f].baseline_latency_ms) for f in eng.functions},
        "counts": {f: [c.arrived, c.completed, c.rejected] for f, c in eng._counts.items()},
        "latencies": {f: [hx(x) for x in v] for f, v in eng._latencies.items()},
        "intervals": [ivd(iv) for iv in eng._intervals],
        "price": hx(eng.cfg.price_per_gpu_hour), "sim_end": hx(sim_end),
        "out": {"violation_curve": {f: [hx(x) for x in v] for f, v in out.violation_curve.items()},
                "percentiles": {f: {k: hx(x) for k, x in v.items()}
                                for f, v in out.percentiles.items()},
                "cost": {f: hx(x) for f, x in out.cost.items()},
                "cost_per_1k": {f: hx(x) for f, x in out.cost_per_1k.items()}}}


def gen_metrics(hs):
    """_finalize inputs/outputs captured from real reference simulations (the demo config,
    three policies) plus synthetic engine states covering the edge cases."""
    import tempfile
    import types
    from hybridscale import cli
    from hybridscale.sim import FunctionCounts, PodCostInterval, SimConfig, SimulationEngine
    records = []
    orig = SimulationEngine._finalize

    def capture(self, sim_end):
        out = orig(self, sim_end)
        records.append(_finalize_record(self, sim_end, out))
        return out
    SimulationEngine._finalize = capture
    try:
        demo = os.path.join(REF_PKG, "configs", "demo.yaml")
        assert cli.main(["run", "--config", demo, "--out", tempfile.mkdtemp()]) == 0
    finally:
        SimulationEngine._finalize = orig
    rng = random.Random(777)
    for case in range(6):
        nf = [3, 1, 5, 2, 4, 8][case]
        fids = [f"fn-{rng.randrange(1000):03d}" for _ in range(nf)]
        fids = list(dict.fromkeys(fids))
        eng = types.SimpleNamespace()
        eng.functions = {f: types.SimpleNamespace(baseline_latency_ms=rng.choice(
            [20.0, 35.5, 12.25, 100.0, 7.0])) for f in fids}
        eng._counts, eng._latencies, eng._intervals = {}, {}, []
        for f in fids:
            n = rng.choice([0, 1, 2, 3, 17, 100, 2500])
            base = eng.functions[f].baseline_latency_ms
            lat = [rng.choice([base * rng.choice([0.5, 1.0, 1.25, 2.0, 9.75, 10.0]),
                               rng.uniform(0, 12 * base), float(rng.randrange(1, 400))])
                   for _ in range(n)]
            rejected = rng.randrange(0, 5)
            unfinished = rng.randrange(0, 3)
            arrived = n + rejected + unfinished if rng.random() > 0.1 or n else 0
            eng._counts[f] = FunctionCounts(arrived=arrived, completed=n,
                                            rejected=rejected if arrived else 0)
            eng._latencies[f] = lat
            for k in range(rng.randrange(0, 6)):
                st = rng.uniform(0, 50000)
                end = -1.0 if rng.random() < 0.3 else st + rng.choice([0.0, rng.uniform(0, 9e4)])
                if rng.random() < 0.1:
                    end = st - 5.0  # negative duration clamps to 0
                eng._intervals.append(PodCostInterval(f, f"pod-{k}", "gpu-000",
                                                      rng.randrange(1, 101),
                                                      rng.randrange(1, 101), st, end))
        eng._intervals.append(PodCostInterval("not-managed", "pod-x", "gpu-001", 50, 50, 0.0, 10.0))
        rng.shuffle(eng._intervals)
        eng.cfg = SimConfig(price_per_gpu_hour=rng.choice([2.48, 0.0, 3.1]))
        eng._timeline = []
        sim_end = rng.uniform(60000, 200000)
        out = SimulationEngine._finalize(eng, sim_end)
        records.append(_finalize_record(eng, sim_end, out))
    dump("metrics.json", records)


# -- trace replay: real simulator runs, captured at every scaler tick ------------------------


def _replay_capture(hs, eng, name):
    """Runs the engine, recording per tick what a batched _handle_scaler needs: arrivals,
    idle pods, pods released by completions since the last tick, and the outcome."""
    from hybridscale.sim import SimulationEngine
    rec = {"name": name, "ticks": []}
    state = {"in_tick": False, "released": [], "first": True}
    orig_release = eng._release_pod
    orig_handle = eng._handle_scaler
    recorded = []
    orig_decide = eng.policy.decide

    def spy_decide(function, cl, rate):
        acts = orig_decide(function, cl, rate)
        recorded.extend(acts)
        return acts

    def spy_release(pod_id, now):
        if not state["in_tick"]:
            state["released"].append(pod_id)
        return orig_release(pod_id, now)

    def spy_handle(now):
        if state["first"]:
            state["first"] = False
            rec["initial"] = cluster_dict(eng.cluster)
            rec["pod_counter0"] = eng._pod_counter
            state["released"].clear()
        fids = sorted(eng.functions)
        arrivals = [eng._tick_arrivals[f] for f in fids]
        idle = sorted(pid for pid, rt in eng._runtimes.items() if rt.idle())
        ready = sorted([pid, hx(rt.pod.ready_at_ms)] for pid, rt in eng._runtimes.items()
                       if rt.pod.state.value == "cold_starting")
        released = list(state["released"])
        state["released"].clear()
        recorded.clear()
        n_before = eng._pod_counter
        state["in_tick"] = True
        orig_handle(now)
        state["in_tick"] = False
        tl = eng._timeline[-len(fids):]
        rec["ticks"].append({
            "now": hx(now), "arrivals": arrivals, "idle": idle, "released": released,
            "cold": ready, "actions": action_list(recorded),
            "new_pods": [f"pod-{i:06d}" for i in range(n_before, eng._pod_counter)],
            "observed": [hx(p.observed_rps) for p in tl],
            "predicted": [hx(p.predicted_rps) for p in tl]})

    eng._release_pod = spy_release
    eng._handle_scaler = spy_handle
    eng.policy.decide = spy_decide
    eng.run()
    rec["trailing_released"] = list(state["released"])  # completions after the last tick
    rec["final"] = cluster_dict(eng.cluster)
    return rec


def gen_replay(hs):
    """Config-3-style trace replays through the reference simulator: the demo experiment
    (2 functions, step-burst trace, all three policies) and a 100-function burst replay on
    64 GPUs (hybrid).  Tables, functions and configs are stored with the captures."""
    from hybridscale import (FunctionSpec, PerfTable, PodConfig, ScalerConfig, SimConfig,
                             build_cluster, load_table)
    from hybridscale.sim import SimulationEngine
    from hybridscale.trace import merge_traces, synth_trace
    runs = []
    # 1) the demo experiment (pkg/configs/demo.yaml) built through the reference's own API
    tables = {n: load_table(os.path.join(REF_PKG, "tables", n + ".csv"))
              for n in ("resnet50", "bert-small")}
    fdefs = [("resnet50", 20.0, [1, 2, 4, 8], PodConfig(8, 75, 20, 1)),
             ("bert-small", 29.0, [1, 2, 4], PodConfig(4, 75, 20, 1))]
    trace = merge_traces([
        synth_trace("step", {"low": 20, "high": 200, "period_ms": 60000}, 42,
                    function_id="resnet50", horizon_ms=240000.0),
        synth_trace("step", {"low": 10, "high": 60, "period_ms": 60000}, 43,
                    function_id="bert-small", horizon_ms=240000.0)])
    kal = {"A": 1.0, "Q": 25.0, "H": 1.0, "D": 4.0, "P0": 1.0}
    for policy in ("hybrid", "horizontal-only", "exclusive-gpu"):
        fns = [FunctionSpec(function_id=f, baseline_latency_ms=bl, perf_table_ref=f,
                            min_rps=1.0, allowed_batches=ab, initial=ini)
               for f, bl, ab, ini in fdefs]
        cluster = build_cluster(4, functions=fns, total_sm_units=80)
        cfg = ScalerConfig(alpha=0.65, beta=0.45, delta_iq=10, cooldown_ms=30000.0, r_min=1.0)
        simcfg = SimConfig(window_ms=100.0, scaler_interval_ms=1000.0, cold_start_ms=5000.0,
                           queue_capacity=1000, seed=42)
        eng = SimulationEngine(trace, fns, tables, cluster, cfg, simcfg, policy, kal)
        rec = _replay_capture(hs, eng, f"demo-{policy}")
        rec.update({"policy": policy, "functions": [fn_dict(f) for f in fns],
                    "tables": {n: table_dict(t) for n, t in tables.items()},
                    "alpha": hx(0.65), "beta": hx(0.45), "delta": 10,
                    "cooldown_ms": hx(30000.0), "r_min": hx(1.0), "interval_ms": hx(1000.0),
                    "cold_start_ms": hx(5000.0), "kalman": {k: hx(v) for k, v in kal.items()}})
        runs.append(rec)
    # 2) 100 functions, burst traces, 64 GPUs (BASELINE config 3), hybrid
    rng = random.Random(3)
    fns, tables, traces = [], {}, []
    bs, ss, qs = [1, 2, 4, 8, 16, 32], list(range(10, 101, 10)), list(range(10, 101, 10))
    for i in range(100):
        fid = f"fn-{i:03d}"
        fixed, per, floor = rng.uniform(4, 20), rng.uniform(0.5, 4), rng.uniform(0.2, 0.4)
        lat = np.array([[[(fixed + per * b) * (floor + (1.0 - floor) * (100.0 / s)) * (100.0 / q)
                          for q in qs] for s in ss] for b in bs])
        tables[fid] = PerfTable(fid, bs, ss, qs, lat)
        fns.append(FunctionSpec(function_id=fid, baseline_latency_ms=20.0, perf_table_ref=fid,
                                min_rps=1.0, allowed_batches=[1, 2, 4, 8],
                                initial=PodConfig(4, rng.choice([20, 30, 40]), 20, 1)))
        traces.append(synth_trace("burst", {"base": rng.uniform(2, 20),
                                            "spike": rng.uniform(40, 120), "spike_prob": 0.2},
                                  1000 + i, function_id=fid, horizon_ms=60000.0))
    trace = merge_traces(traces)
    cluster = build_cluster(64, functions=fns)
    cfg = ScalerConfig(alpha=0.65, beta=0.45, delta_iq=10, cooldown_ms=5000.0, r_min=1.0)
    simcfg = SimConfig(scaler_interval_ms=1000.0, cold_start_ms=2000.0, queue_capacity=1000,
                       seed=7, max_drain_ms=5000.0)
    eng = SimulationEngine(trace, fns, tables, cluster, cfg, simcfg, "hybrid", kal)
    rec = _replay_capture(hs, eng, "burst-100")
    rec.update({"policy": "hybrid", "functions": [fn_dict(f) for f in fns],
                "tables": {n: table_dict(t) for n, t in tables.items()},
                "alpha": hx(0.65), "beta": hx(0.45), "delta": 10, "cooldown_ms": hx(5000.0),
                "r_min": hx(1.0), "interval_ms": hx(1000.0), "cold_start_ms": hx(2000.0),
                "kalman": {k: hx(v) for k, v in kal.items()}})
    runs.append(rec)
    dump("replay.json", {"runs": runs})


def _config4_world_ref(hs, nfn, ngpu, seed, full_grid):
    """bench.make_config4_world rebuilt with the reference's own types: the same RNG draws,
    the same gen_tables surfaces (bench.surface), one RUNNING pod (8, 20, 20) per function
    placed round-robin by the reference's allocator."""
    import bench
    from hybridscale import FunctionSpec, PerfTable, PodConfig, PodInstance, PodState, allocator
    from hybridscale.sim import build_cluster
    rng = random.Random(seed)
    if full_grid:
        bs, ss, qs = list(range(1, 33)), list(range(10, 101)), list(range(1, 101))
    else:
        bs, ss, qs = bench.BATCHES, list(range(10, 101, 10)), list(range(10, 101, 10))
    fns, tables, caps = [], {}, {}
    for i in range(nfn):
        fid = f"fn-{i:04d}"
        fixed, per, floor = rng.uniform(4, 20), rng.uniform(0.5, 4), rng.uniform(0.2, 0.4)
        lat = bench.surface(fixed, per, floor, 1.0 - floor, bs, ss, qs)
        tables[fid] = PerfTable(fid, bs, ss, qs, lat)
        fns.append(FunctionSpec(function_id=fid, baseline_latency_ms=20.0, perf_table_ref=fid,
                                allowed_batches=list(bench.BATCHES), initial=PodConfig(8, 20, 20)))
        caps[fid] = 8 / (float(lat[bs.index(8), ss.index(20), qs.index(20)]) / 1000.0)
    cluster = build_cluster(ngpu, functions=fns)
    for i, f in enumerate(fns):
        allocator.place_pod(cluster, PodInstance(f"pod-{i:06d}", f.function_id, 8, 20, 20, "",
                                                 state=PodState.RUNNING), f"gpu-{i % ngpu:03d}")
    return fns, tables, cluster, caps


def gen_config4(hs):
    """BASELINE config 4 through the reference's own SimulationEngine._handle_scaler: 1,000
    functions on 400 GPUs, five ticks of swinging load (the bench's tick workload: interval
    2 s, cold start 5 s, every pod idle, arrivals from bench.config4_arrivals with
    random.Random(0)), in both grid variants (6x10x10 with delta 10; 32x91x100 with delta 1).
    The reference takes minutes per tick here (copy.deepcopy per scale-up)."""
    import time as _time
    import bench
    from hybridscale import ScalerConfig, SimConfig, WorkloadTrace
    from hybridscale.sim import SimulationEngine, _PodRuntime
    variants = [v for v in ("6x10x10", "32x91x100")
                if os.environ.get("GOLDEN_C4_VARIANT", v) == v]
    for variant in variants:
        full = variant != "6x10x10"
        t0 = _time.time()
        fns, tables, cluster, caps = _config4_world_ref(hs, 1000, 400, 0, full)
        cfg = ScalerConfig(delta_iq=1 if full else 10)
        simcfg = SimConfig(scaler_interval_ms=2000.0, cold_start_ms=5000.0)
        eng = SimulationEngine(WorkloadTrace(entries=[], horizon_ms=1.0), fns, tables, cluster,
                               cfg, simcfg, "hybrid", None)
        for pod in cluster.pods.values():  # what _bootstrap does for its own placements
            pod.capability_rps = eng._capability(pod)
            eng._runtimes[pod.pod_id] = _PodRuntime(pod)
            eng._open_cost_interval(pod, 0.0)
        eng._pod_counter = len(cluster.pods)
        recorded = []
        orig = eng.policy.decide

        def spy(function, cl, rate, _orig=orig):
            acts = _orig(function, cl, rate)
            recorded.extend(acts)
            return acts
        eng.policy.decide = spy
        rng = random.Random(0)
        run = {"variant": variant, "nfn": 1000, "ngpu": 400, "seed": 0,
               "delta": cfg.delta_iq, "interval_ms": hx(2000.0), "cold_start_ms": hx(5000.0),
               "pod_counter0": eng._pod_counter, "ticks": []}
        print(f"config4 {variant}: world built in {_time.time() - t0:.0f} s", flush=True)
        for k in range(int(os.environ.get("GOLDEN_C4_TICKS", "5"))):
            now = 2000.0 * (k + 1)
            swing = (1.0, 1.5, 0.2, 2.0, 0.05)[k % 5]
            arrivals = bench.config4_arrivals(fns, caps, rng, 2.0, 0.0, 3.0 * swing)
            for fid, a in arrivals.items():
                eng._tick_arrivals[fid] = a
            for pid, rt in list(eng._runtimes.items()):  # ready events precede the tick
                if rt.pod.state.value == "cold_starting" and rt.pod.ready_at_ms <= now:
                    eng._handle_ready(now, pid)
            recorded.clear()
            n_before = eng._pod_counter
            t1 = _time.time()
            eng._handle_scaler(now)
            tl = eng._timeline[-len(fns):]
            run["ticks"].append({
                "now": hx(now), "arrivals": [arrivals[f.function_id] for f in fns],
                "actions": action_list(recorded),
                "new_pods": [f"pod-{i:06d}" for i in range(n_before, eng._pod_counter)],
                "observed": [hx(p.observed_rps) for p in tl],
                "predicted": [hx(p.predicted_rps) for p in tl],
                "capacity": [hx(p.capacity_rps) for p in tl],
                "reference_s": round(_time.time() - t1, 3)})
            print(f"config4 {variant}: tick {k} {len(recorded)} actions in "
                  f"{_time.time() - t1:.0f} s", flush=True)
        run["final"] = cluster_dict(eng.cluster)
        dump(f"config4_{variant}.json", run)


def _experiments_module():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "rapp_experiments", os.path.join(ROOT, "tests", "experiments.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def gen_csv(hs):
    """sha256 of the four metric CSVs (hs/sim.py:651-685) of pure-reference runs: the demo
    experiment (pkg/configs/demo.yaml, 3 policies) and config 3 (100 functions, 60 s burst
    replay, hybrid and horizontal-only: 100 whole-GPU pods do not fit 64 GPUs).  The GPU tests re-run the same experiments with the B200
    tick and compare bytes (and against a live reference run where the reference is
    installed)."""
    import tempfile
    from hybridscale.sim import run
    ex = _experiments_module()
    out = {}
    specs = ex.demo_runs(hs, os.path.join(REF_PKG, "configs", "demo.yaml")) + \
        ex.config3_runs(hs, policies=("hybrid", "horizontal-only"))
    for spec in specs:
        with tempfile.TemporaryDirectory() as d:
            out[spec[0]] = ex.digest(ex.run_to_csvs(run, spec, d))
        print(spec[0], out[spec[0]]["timeline.csv"], flush=True)
    dump("csv.json", out)


GENERATORS = {"interp": gen_interp, "mec": gen_mec, "scale": gen_scale, "tick": gen_tick,
              "policy": gen_policy, "ingest": gen_ingest,
              "metrics": gen_metrics, "replay": gen_replay, "config4": gen_config4,
              "csv": gen_csv}


def main(argv):
    hs = import_reference()
    names = argv or list(GENERATORS)
    for name in names:
        GENERATORS[name](hs)


if __name__ == "__main__":
    main(sys.argv[1:])
