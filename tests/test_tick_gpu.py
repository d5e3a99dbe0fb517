"""The batched device tick vs the real reference (golden decisions and ticks) and vs the
scaler oracle on config-4-sized ticks.  Mirrors pkg/tests/test_autoscaler.py,
test_acceptance.py C2 and the sim's per-tick loop (hs/sim.py:470-491)."""

import copy
import random

import numpy as np
import pytest

from oracle import scaler_oracle as so

from .conftest import golden_table_arrays, load_golden
from .golden_io import (cluster_from, cluster_to, function_from, fx, golden_cluster_to,
                        make_part, make_pod, surface_tables)

pytestmark = pytest.mark.gpu


def _cfg_obj(c):
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    a, b, d, cd, rmin = c
    return ScalerConfig(alpha=fx(a), beta=fx(b), delta_iq=d, cooldown_ms=fx(cd), r_min=fx(rmin))


def _acts(actions):
    return [[a.function_id, a.kind.value, a.batch, a.sm_percent, a.quota_percent, a.pod_id,
             a.gpu_id] for a in actions]


def test_scale_matches_reference_golden():
    """Every single-function decision of the reference (1,610 cases incl. the six
    hand-traced conformance scenarios and the three randomized loops)."""
    from paper_2505_01968_b200 import PerfTable
    from paper_2505_01968_b200.autoscaler import Autoscaler
    g = load_golden("scale.json")
    t = g["table"]
    b, s, q, v = golden_table_arrays(t)
    table = PerfTable(t["function_id"], t["batches"], t["sms"], t["quotas"], v)
    fn = function_from(g["function"])
    for case in g["cases"]:
        sc = Autoscaler(_cfg_obj(case["cfg"]), {"conf-fn": table})
        if case["last_down"] is not None:
            sc._last_scale_down["conf-fn"] = fx(case["last_down"])
        cluster = cluster_from(case["cluster"])
        got = _acts(sc.scale(fn, cluster, fx(case["rate"])))
        assert got == case["actions"], case["name"]
        want_stamp = fx(case["stamp"])
        assert sc._last_scale_down.get("conf-fn") == want_stamp, case["name"]
        assert cluster_to(cluster) == golden_cluster_to(case["cluster"]), case["name"]


def _engine_for_run(run, apply_to_host=True):
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    from paper_2505_01968_b200.tick import TickEngine
    fns = [function_from(f) for f in run["functions"]]
    tables = surface_tables(run["tables"], fns)
    cluster = cluster_from(run["initial"])
    cfg = ScalerConfig(alpha=fx(run["alpha"]), beta=fx(run["beta"]), delta_iq=run["delta"],
                       cooldown_ms=fx(run["cooldown_ms"]), r_min=fx(run["r_min"]))
    kal = {k: fx(v) for k, v in run["kalman"].items()}
    eng = TickEngine(fns, tables, cluster, cfg, kalman_params=kal,
                     scaler_interval_ms=fx(run["interval_ms"]),
                     cold_start_ms=fx(run["cold_start_ms"]), pod_counter=run["pod_counter0"],
                     policy=run.get("policy", "hybrid"))
    return eng, fns, cluster


def test_ticks_match_reference_golden():
    """Multi-tick runs of the reference's _handle_scaler (Kalman, decisions, apply with new
    pod ids, releases of idle drained pods, cold-start promotion), 0-ulp rates."""
    g = load_golden("tick.json")
    for run in g["runs"]:
        eng, fns, cluster = _engine_for_run(run)
        fids = [f["id"] for f in run["functions"]]
        for t in run["ticks"]:
            res = eng.tick(fx(t["now"]), t["arrivals"], idle=set(t["idle"]), apply_to_host=True)
            assert _acts(res.actions) == [list(a) for a in t["actions"]]
            assert [a for a, k in zip(res.pod_ids, res.actions)
                    if k.kind.value == "horizontal_up"] == t["new_pods"]
            assert [res.observed[f] for f in fids] == [fx(x) for x in t["observed"]]
            assert [res.predicted[f] for f in fids] == [fx(x) for x in t["predicted"]]
            cluster.validate()
        assert cluster_to(cluster) == golden_cluster_to(run["final"])
        # the device world agrees with the host mirror
        dev = eng.device_cluster_dict()
        host = cluster_to(cluster)
        assert dev["pods"] == sorted(host["pods"], key=str)
        for gpu in host["gpus"]:
            assert [(p["sm"], p["alloc"], len(p["residents"])) for p in gpu["partitions"]] == \
                dev["partitions"][gpu["id"]]


def _oracle_ticks(fns, tables, cluster, cfg, nticks, seed, interval_ms=2000.0,
                  cold_start_ms=5000.0, kal=None):
    """Runs the oracle and the device engine side by side on the same inputs."""
    from paper_2505_01968_b200.tick import TickEngine
    import bench
    kal = kal or {"A": 1.0, "Q": 4.0, "H": 1.0, "D": 16.0, "P0": 1.0}
    eng = TickEngine(fns, tables, copy.deepcopy(cluster), cfg, kalman_params=kal,
                     scaler_interval_ms=interval_ms, cold_start_ms=cold_start_ms,
                     pod_counter=len(cluster.pods))
    ocl = copy.deepcopy(cluster)
    otables = {k: so.OTable(t) for k, t in tables.items()}
    ocfg = {"alpha": cfg.alpha, "beta": cfg.beta, "delta": cfg.delta_iq,
            "cooldown_ms": cfg.cooldown_ms, "r_min": cfg.r_min}
    okal = {k: v for k, v in kal.items() if k != "P0"}
    kstate, last_down = {}, {}
    counter = len(cluster.pods)
    functions = {f.function_id: f for f in fns}
    caps = {f.function_id: otables[f.function_id].thr(8, 20, 20) for f in fns}
    rng = random.Random(seed)
    n_actions = 0
    for k in range(nticks):
        now = interval_ms * (k + 1)
        swing = (1.0, 1.5, 0.2, 2.0, 0.05)[k % 5]
        arrivals = bench.config4_arrivals(fns, caps, rng, interval_ms / 1000.0, 0.0, 3.0 * swing)
        idle = {pid for pid in eng.pod_ids if rng.random() < 0.7}
        acts, obs, pred, counter = so.tick(ocfg, functions, otables, ocl, now, interval_ms,
                                           arrivals, idle, kstate, okal, kal["P0"], last_down,
                                           counter, make_pod, make_part,
                                           cold_start_ms=cold_start_ms)
        res = eng.tick(now, arrivals, idle=idle)
        got = [[a.function_id, a.kind.value, a.batch, a.sm_percent, a.quota_percent, pid,
                a.gpu_id] for a, pid in zip(res.actions, res.pod_ids)]
        assert got == [list(a) for a in acts], f"tick {k}"
        assert res.predicted == pred and res.observed == obs
        n_actions += len(acts)
    dev = eng.device_cluster_dict()
    assert dev["pods"] == sorted(cluster_to(ocl)["pods"], key=str)
    return n_actions


@pytest.mark.parametrize("variant", ["6x10x10", "32x91x100"])
def test_config4_ticks_match_reference(variant):
    """BASELINE config 4 pinned to the reference itself: 1,000 functions on 400 GPUs, the
    bench's five swinging-load ticks, captured from hybridscale's own
    SimulationEngine._handle_scaler (tests/golden/gen_golden.py gen_config4) — both grid
    variants (6x10x10 tables with delta 10; 32x91x100 tables with delta 1, whose fresh-GPU
    searches run on 54,600-point lattices).  Identical ordered action lists, new pod ids,
    0-ulp observed / predicted rates and the same final cluster."""
    import bench
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    from paper_2505_01968_b200.tick import TickEngine
    g = load_golden(f"config4_{variant}.json")
    fns, tables, cluster, _ = bench.make_config4_world(g["nfn"], g["ngpu"], seed=g["seed"],
                                                       full_grid=variant != "6x10x10")
    eng = TickEngine(fns, tables, cluster, ScalerConfig(delta_iq=g["delta"]),
                     scaler_interval_ms=fx(g["interval_ms"]),
                     cold_start_ms=fx(g["cold_start_ms"]), pod_counter=g["pod_counter0"])
    fids = sorted(f.function_id for f in fns)
    for k, t in enumerate(g["ticks"]):
        res = eng.tick(fx(t["now"]), t["arrivals"], idle=None, apply_to_host=True)
        assert _acts(res.actions) == [list(a) for a in t["actions"]], f"tick {k}"
        assert [p for p, a in zip(res.pod_ids, res.actions)
                if a.kind.value == "horizontal_up"] == t["new_pods"], f"tick {k}"
        assert [res.observed[f] for f in fids] == [fx(x) for x in t["observed"]]
        assert [res.predicted[f] for f in fids] == [fx(x) for x in t["predicted"]]
    assert cluster_to(cluster) == golden_cluster_to(g["final"])


def test_config4_ticks_vs_oracle():
    """1,000 functions on 400 GPUs (config 4), five ticks with swinging load."""
    import bench
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    fns, tables, cluster, _ = bench.make_config4_world(1000, 400, seed=0)
    n = _oracle_ticks(fns, tables, cluster, ScalerConfig(), 5, seed=1)
    assert n > 1000


@pytest.mark.parametrize("delta,ngpu,nfn", [(1, 50, 60), (7, 30, 80), (25, 200, 150),
                                            (10, 12, 40), (2, 120, 300), (4, 60, 200),
                                            (1, 200, 100), (3, 300, 150)])
def test_random_worlds_vs_oracle(delta, ngpu, nfn):
    """Quota steps 1..25, crowded and sparse clusters (fresh-GPU branch, releases).  With
    quota steps <= 4 phase A2 tabulates only the tick-start slot sms; the shares left beside
    fresh-GPU placements (100 - s, s on the table's 10% grid) and freed by releases are
    evaluated by the commit from A2's brackets."""
    import bench
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    fns, tables, cluster, _ = bench.make_config4_world(nfn, ngpu, seed=delta)
    cfg = ScalerConfig(alpha=0.85, beta=0.4, delta_iq=delta, cooldown_ms=1000.0, r_min=1.0)
    _oracle_ticks(fns, tables, cluster, cfg, 8, seed=delta, interval_ms=1000.0,
                  cold_start_ms=1500.0)


def test_many_gpus_global_summaries_vs_oracle():
    """6,000 / 9,000 GPUs: the partition lists, then also the per-GPU summaries, no longer
    fit the commit's shared-memory budget, so the commit runs on global memory (and without
    straight-line runs); ids past gpu-999 also exercise string-ordered GPU ranks."""
    import bench
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    for ngpu in (6000, 9000):  # summaries in shared memory without partition lists; neither
        fns, tables, cluster, _ = bench.make_config4_world(48, ngpu, seed=11)
        cfg = ScalerConfig(alpha=0.85, beta=0.4, delta_iq=10, cooldown_ms=1000.0, r_min=1.0)
        _oracle_ticks(fns, tables, cluster, cfg, 4, seed=11, interval_ms=1000.0,
                      cold_start_ms=1500.0)


def test_full_grid_fresh_gpu_search_vs_oracle():
    """Full-grid tables (32x91x100, delta 1): the fresh-GPU most_efficient_config runs on a
    291,200-point lattice through the prefix-max index."""
    import bench
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    fns, tables, cluster, _ = bench.make_config4_world(12, 40, seed=3, full_grid=True)
    cfg = ScalerConfig(alpha=0.9, beta=0.5, delta_iq=1, cooldown_ms=1000.0, r_min=1.0)
    _oracle_ticks(fns, tables, cluster, cfg, 4, seed=5, interval_ms=1000.0,
                  cold_start_ms=1500.0)


@pytest.mark.parametrize("delta,ngpu,nfn,full", [(1, 50, 60, False), (2, 120, 300, False),
                                                 (4, 60, 200, False), (1, 60, 40, True)])
def test_bracket_rows_vs_oracle(monkeypatch, delta, ngpu, nfn, full):
    """RAPP_TICK_MASK_NONE=1 makes phase A2 tabulate no row, so every used-GPU placement reads
    its throughput row through the commit's bracket path (the path of slot shares outside
    the tick-start mask, rare in these worlds) — decisions must still equal the oracle."""
    import bench
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    monkeypatch.setenv("RAPP_TICK_MASK_NONE", "1")
    fns, tables, cluster, _ = bench.make_config4_world(nfn, ngpu, seed=delta + 40,
                                                       full_grid=full)
    cfg = ScalerConfig(alpha=0.85, beta=0.4, delta_iq=delta, cooldown_ms=1000.0, r_min=1.0)
    _oracle_ticks(fns, tables, cluster, cfg, 6, seed=delta + 41, interval_ms=1000.0,
                  cold_start_ms=1500.0)


def test_replica_policies_match_reference_golden():
    """horizontal-only / exclusive-gpu decisions (hs/policies.py:69-141), 1,800 cases."""
    from paper_2505_01968_b200 import PerfTable
    from paper_2505_01968_b200.core import FunctionSpec, PodConfig
    from paper_2505_01968_b200.policies import make_policy
    g = load_golden("policy.json")
    t = g["table"]
    b, s, q, v = golden_table_arrays(t)
    table = PerfTable(t["function_id"], t["batches"], t["sms"], t["quotas"], v)
    for case in g["cases"]:
        fn = FunctionSpec("conf-fn", 20.0, perf_table_ref="conf-fn", allowed_batches=[8],
                          initial=PodConfig(*case["initial"]))
        pol = make_policy(case["policy"], _cfg_obj(case["cfg"]), {"conf-fn": table})
        if case["last_down"] is not None:
            pol._last_scale_down["conf-fn"] = fx(case["last_down"])
        got = _acts(pol.decide(fn, cluster_from(case["cluster"]), fx(case["rate"])))
        assert got == case["actions"]
        assert pol._last_scale_down.get("conf-fn") == fx(case["stamp"])


def test_policy_hand_cases():
    """pkg/tests/test_policies.py: 4 fixed-shape replicas packed onto gpu-000; newest-first
    removal; never the last pod; whole-GPU replicas need a free GPU; aliases."""
    from paper_2505_01968_b200 import PerfTable
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    from paper_2505_01968_b200.core import (ClusterState, FunctionSpec, GpuDevice, PodConfig,
                                            PodInstance, PodState)
    from bench import place_initial
    from paper_2505_01968_b200.errors import ConfigError
    from paper_2505_01968_b200.policies import (ExclusiveGpuPolicy, HorizontalOnlyPolicy,
                                                make_policy)
    quotas = list(range(10, 101, 10))
    lat = np.zeros((1, 2, 10))
    for qi, qq in enumerate(quotas):
        lat[0, 1, qi] = 8000.0 / (2.0 * qq + 10.0)
        lat[0, 0, qi] = 2.0 * lat[0, 1, qi]
    tables = {"conf-fn": PerfTable("conf-fn", [8], [25, 50], quotas, lat)}
    cfg = ScalerConfig(alpha=0.9, beta=0.5, delta_iq=20)
    fn = FunctionSpec("conf-fn", 20.0, perf_table_ref="conf-fn", allowed_batches=[8],
                      initial=PodConfig(8, 50, 20))

    def cluster(n):
        return ClusterState(gpus={f"gpu-{i:03d}": GpuDevice(f"gpu-{i:03d}") for i in range(n)})

    def put(c, pid, sm, qq, gpu):
        place_initial(c, PodInstance(pid, "conf-fn", 8, sm, qq, gpu,
                                     state=PodState.RUNNING), gpu)

    assert isinstance(make_policy("horizontal", cfg, tables), HorizontalOnlyPolicy)
    assert isinstance(make_policy("exclusive", cfg, tables), ExclusiveGpuPolicy)
    with pytest.raises(ConfigError):
        make_policy("magic", cfg, tables)
    c = cluster(3)
    put(c, "p0", 50, 20, "gpu-000")
    acts = make_policy("horizontal-only", cfg, tables).decide(fn, c, 200.0)
    assert [(a.kind.value, a.batch, a.sm_percent, a.quota_percent, a.gpu_id) for a in acts] == \
        [("horizontal_up", 8, 50, 20, "gpu-000")] * 4
    c = cluster(2)
    for i in range(3):
        put(c, f"p{i}", 50, 20, "gpu-000")
    c.clock_ms = 60_000.0
    pol = make_policy("horizontal-only", cfg, tables)
    assert [a.pod_id for a in pol.decide(fn, c, 20.0)] == ["p2", "p1"]
    c.clock_ms = 70_000.0
    assert pol.decide(fn, c, 20.0) == []  # cooldown
    c = cluster(1)
    put(c, "p0", 50, 20, "gpu-000")
    c.clock_ms = 60_000.0
    assert make_policy("horizontal-only", cfg, tables).decide(fn, c, 2.0) == []
    c = cluster(2)
    put(c, "p0", 100, 100, "gpu-000")
    acts = make_policy("exclusive-gpu", cfg, tables).decide(fn, c, 2000.0)
    assert [(a.gpu_id, a.sm_percent, a.quota_percent) for a in acts] == [("gpu-001", 100, 100)]


@pytest.mark.parametrize("policy", ["horizontal-only", "exclusive-gpu"])
def test_replica_ticks_vs_oracle_at_scale(policy):
    """300 functions, replica policies, several ticks: device vs oracle."""
    import bench
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    from paper_2505_01968_b200.tick import TickEngine
    fns, tables, cluster, _ = bench.make_config4_world(300, 400, seed=11)
    cfg = ScalerConfig(alpha=0.8, beta=0.4, delta_iq=10, cooldown_ms=1000.0)
    eng = TickEngine(fns, tables, copy.deepcopy(cluster), cfg, scaler_interval_ms=1000.0,
                     cold_start_ms=1500.0, pod_counter=300, policy=policy)
    ocl = copy.deepcopy(cluster)
    otables = {k: so.OTable(t) for k, t in tables.items()}
    ocfg = {"alpha": 0.8, "beta": 0.4, "delta": 10, "cooldown_ms": 1000.0, "r_min": 1.0}
    kal = {"A": 1.0, "Q": 4.0, "H": 1.0, "D": 16.0}
    kstate, last, counter = {}, {}, 300
    functions = {f.function_id: f for f in fns}
    caps = {f.function_id: otables[f.function_id].thr(8, 20, 20) for f in fns}
    rng = random.Random(4)
    total = 0
    for k in range(6):
        now = 1000.0 * (k + 1)
        arr = bench.config4_arrivals(fns, caps, rng, 1.0, 0.0, (4.0, 0.1, 3.0, 0.02, 5.0, 0.3)[k])
        idle = {pid for pid in eng.pod_ids if rng.random() < 0.6}
        acts, obs, pred, counter = so.tick(ocfg, functions, otables, ocl, now, 1000.0, arr, idle,
                                           kstate, kal, 1.0, last, counter, make_pod, make_part,
                                           cold_start_ms=1500.0, policy=policy)
        res = eng.tick(now, arr, idle=idle)
        got = [[a.function_id, a.kind.value, a.batch, a.sm_percent, a.quota_percent, pid,
                a.gpu_id] for a, pid in zip(res.actions, res.pod_ids)]
        assert got == [list(a) for a in acts], f"tick {k}"
        total += len(acts)
    assert total > 50


def test_trace_replay_matches_reference_simulator():
    """Every scaler tick of real reference simulations (the demo experiment under all three
    policies, 240 ticks each, and a 100-function burst replay on 64 GPUs): the device tick
    fed the simulator's arrivals, idle pods and between-tick releases makes the same
    decisions, creates the same pod ids and reports the same rates (0 ulp)."""
    from paper_2505_01968_b200 import PerfTable
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    from paper_2505_01968_b200.tick import TickEngine
    g = load_golden("replay.json")
    for run in g["runs"]:
        fns = [function_from(f) for f in run["functions"]]
        tables = {}
        for name, t in run["tables"].items():
            b, s, q, v = golden_table_arrays(t)
            tables[name] = PerfTable(t["function_id"], t["batches"], t["sms"], t["quotas"], v)
        cluster = cluster_from(run["initial"])
        cfg = ScalerConfig(alpha=fx(run["alpha"]), beta=fx(run["beta"]), delta_iq=run["delta"],
                           cooldown_ms=fx(run["cooldown_ms"]), r_min=fx(run["r_min"]))
        eng = TickEngine(fns, tables, cluster, cfg,
                         kalman_params={k: fx(v) for k, v in run["kalman"].items()},
                         scaler_interval_ms=fx(run["interval_ms"]),
                         cold_start_ms=fx(run["cold_start_ms"]),
                         pod_counter=run["pod_counter0"], policy=run["policy"])
        fids = sorted(f["id"] for f in run["functions"])
        for k, t in enumerate(run["ticks"]):
            eng.release(t["released"], apply_to_host=True)
            res = eng.tick(fx(t["now"]), t["arrivals"], idle=set(t["idle"]),
                           apply_to_host=True)
            assert _acts(res.actions) == [list(a) for a in t["actions"]], (run["name"], k)
            assert [a for a, x in zip(res.pod_ids, res.actions)
                    if x.kind.value == "horizontal_up"] == t["new_pods"], (run["name"], k)
            assert [res.observed[f] for f in fids] == [fx(x) for x in t["observed"]]
            assert [res.predicted[f] for f in fids] == [fx(x) for x in t["predicted"]]
            cluster.validate()
        eng.release(run["trailing_released"], apply_to_host=True)
        assert cluster_to(cluster) == golden_cluster_to(run["final"]), run["name"]
        dev = eng.device_cluster_dict()
        assert dev["pods"] == sorted(cluster_to(cluster)["pods"], key=str), run["name"]
