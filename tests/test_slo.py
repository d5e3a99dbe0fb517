"""Opt-in latency <= SLO feasibility mask (north_star (3); an extension: the reference
never reads FunctionSpec.slo_ms, hs/core.py:96-98, and searches on rps >= target only,
hs/perf.py:132).  CPU: the restatement (oracle/slo_oracle.py) reduces to the pinned oracle
and the reference's golden answers when the SLO cannot bind.  GPU: the lattice kernel
(rapp_mec_plan_set_slo) and the tick's fresh-GPU search (rapp_tick_set_slo) against the
restatement, and the default (no SLO) path unchanged."""

import copy
import math

import numpy as np
import pytest

from .conftest import golden_table_arrays
from oracle.slo_oracle import OTableSLO, mec_slo


def test_slo_restatement_reduces_to_reference_rule(mec_golden):
    tables = {t["function_id"]: golden_table_arrays(t) for t in mec_golden["tables"]}
    for case in mec_golden["cases"][::7]:
        b, s, q, v = tables[case["table"]]
        got = mec_slo(b, s, q, v, float.fromhex(case["target"]), case["step"], case["batches"],
                      math.inf)
        assert list(got) == case["result"], case


def _tables(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        fixed, per, floor = rng.uniform(4, 20), rng.uniform(0.5, 4), rng.uniform(0.2, 0.4)
        b = np.array([1.0, 2.0, 4.0, 8.0, 16.0, 32.0])
        s = np.arange(10.0, 101.0, 10.0)
        q = np.arange(10.0, 101.0, 10.0)
        v = ((fixed + per * b)[:, None, None] * (floor + (1 - floor) * (100.0 / s))[None, :, None]
             * (100.0 / q)[None, None, :])
        out.append((b, s, q, np.ascontiguousarray(v)))
    return out


def test_slo_restatement_semantics():
    """Every answer meets both bounds when one does; a binding SLO never answers with a
    point whose latency exceeds it unless nothing is feasible (then: max rps overall)."""
    from oracle.binding import or_interp3
    for b, s, q, v in _tables(4, 3):
        top = 32.0 / (v[-1, -1, -1] / 1000.0)
        for target in (0.01 * top, 0.3 * top, 0.9 * top):
            for slo in (5.0, 40.0, 200.0, 1e9):
                bb, ss, qq = mec_slo(b, s, q, v, target, 10, None, slo)
                lat = or_interp3(b, s, q, v, float(bb), float(ss), float(qq))
                rps = bb / (lat / 1000.0)
                if not (rps >= target and lat <= slo):
                    # nothing feasible: the reference's fallback = max throughput
                    assert (bb, ss, qq) == mec_slo(b, s, q, v, 1e300, 10, None, math.inf)


@pytest.mark.gpu
def test_slo_lattice_kernel_vs_restatement():
    from paper_2505_01968_b200 import PerfTable, PerfTableSet
    tabs = _tables(12, 5)
    pts = [PerfTable(f"f{i}", b.astype(int).tolist(), s.astype(int).tolist(),
                     q.astype(int).tolist(), v) for i, (b, s, q, v) in enumerate(tabs)]
    rng = np.random.default_rng(9)
    for step in (1, 10, 20):
        allowed = [None, [2, 4, 8], [1, 3, 5, 32]]
        funcs = [(t, allowed[i % 3]) for i, t in enumerate(pts)]
        ts = PerfTableSet(funcs, quota_step=step)
        base = None
        for rep in range(4):
            targets = [float(rng.uniform(0.5, 1.2) * 32.0 / (t.latency_ms[-1, -1, -1] / 1000.0)
                             * rng.choice([0.01, 0.2, 0.6, 1.0])) for t in pts]
            slos = [None if i % 5 == 0 else float(rng.choice([3.0, 12.0, 40.0, 150.0, 1e6]))
                    for i in range(len(pts))]
            if base is None:  # default path first: the reference rule
                base = ts.search(targets)
                want0 = [mec_slo(t._b_axis, t._s_axis, t._q_axis, t.latency_ms, tg, step, al,
                                 None) for (t, al), tg in zip(funcs, targets)]
                assert base == want0
            ts.set_slo(slos)
            got = ts.search(targets)
            want = [mec_slo(t._b_axis, t._s_axis, t._q_axis, t.latency_ms, tg, step, al, sl)
                    for (t, al), tg, sl in zip(funcs, targets, slos)]
            assert got == want, (step, rep)
            ts.set_slo(None)
            assert ts.search(targets) == [
                mec_slo(t._b_axis, t._s_axis, t._q_axis, t.latency_ms, tg, step, al, None)
                for (t, al), tg in zip(funcs, targets)]
        # the scalar API
        t = pts[0]
        for slo in (4.0, 30.0, None):
            for tg in (1.0, 100.0, 1e7):
                assert t.most_efficient_config(tg, quota_step=step, slo_ms=slo) == mec_slo(
                    t._b_axis, t._s_axis, t._q_axis, t.latency_ms, tg, step, None, slo)
    with pytest.raises(ValueError):
        PerfTableSet([(pts[0], None)], slo_ms=[0.0])


def saturated_world(nfn, ngpu, seed=4):
    """nfn functions with gen_tables surfaces, one pod each at (b=8, s=50, q=100), two per
    GPU (their GPUs' SM and quota are fully allocated), then free GPUs: every scale-up
    needs the fresh-GPU most_efficient_config (hs/autoscaler.py:155-165)."""
    import random
    from bench import BATCHES, place_initial, surface
    from paper_2505_01968_b200 import PerfTable
    from paper_2505_01968_b200.core import (ClusterState, FunctionSpec, GpuDevice, PodConfig,
                                            PodInstance, PodState)
    rng = random.Random(seed)
    ss = qs = list(range(10, 101, 10))
    fns, tables, caps = [], {}, {}
    for i in range(nfn):
        fid = f"fn-{i:04d}"
        fixed, per, floor = rng.uniform(4, 20), rng.uniform(0.5, 4), rng.uniform(0.2, 0.4)
        lat = surface(fixed, per, floor, 1.0 - floor, BATCHES, ss, qs)
        tables[fid] = PerfTable(fid, BATCHES, ss, qs, lat)
        fns.append(FunctionSpec(function_id=fid, baseline_latency_ms=20.0, perf_table_ref=fid,
                                allowed_batches=list(BATCHES), initial=PodConfig(8, 50, 100)))
        caps[fid] = 8 / (float(lat[BATCHES.index(8), ss.index(50), -1]) / 1000.0)
    cluster = ClusterState(gpus={f"gpu-{g:03d}": GpuDevice(f"gpu-{g:03d}") for g in range(ngpu)},
                           functions={f.function_id: f for f in fns})
    for i, f in enumerate(fns):
        place_initial(cluster, PodInstance(f"pod-{i:06d}", f.function_id, 8, 50, 100, "",
                                           state=PodState.RUNNING), f"gpu-{i // 2:03d}")
    return fns, tables, cluster, caps


@pytest.mark.gpu
@pytest.mark.parametrize("mult", [0.9, 2.0, 6.0])
def test_slo_tick_fresh_gpu_search_vs_oracle(mult):
    """Swinging-load ticks of a world whose functions scale onto fresh GPUs: with
    slo_mask=True every fresh-GPU configuration obeys the function's slo_ms (baseline
    latency x multiplier) exactly as the restatement decides it; everything else is the
    reference procedure (oracle/scaler_oracle.py)."""
    import random
    from oracle import scaler_oracle as so
    from bench import config4_arrivals
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    from paper_2505_01968_b200.core import PodInstance, PodState, SmPartition
    from paper_2505_01968_b200.tick import TickEngine
    fns, tables, cluster, caps = saturated_world(24, 40)
    for f in fns:  # SLO = mult x the function's fastest batch-8 latency (s = q = 100)
        f.baseline_latency_ms = float(tables[f.function_id].latency_ms[3, -1, -1]) * mult
        f.slo_multiplier = 1.0
    cfg = ScalerConfig(delta_iq=10)
    ocl = copy.deepcopy(cluster)
    plain = TickEngine(fns, tables, copy.deepcopy(cluster), cfg, scaler_interval_ms=2000.0,
                       cold_start_ms=5000.0, pod_counter=len(fns))
    eng = TickEngine(fns, tables, cluster, cfg, scaler_interval_ms=2000.0, cold_start_ms=5000.0,
                     pod_counter=len(fns), slo_mask=True)
    differs = 0
    otables = {k: OTableSLO(t, next(f.slo_ms for f in fns if f.function_id == k))
               for k, t in tables.items()}
    functions = {f.function_id: f for f in fns}
    rng = random.Random(1)
    kstate, last_down, counter = {}, {}, len(fns)
    fresh = 0
    for k in range(6):
        arr = config4_arrivals(fns, caps, rng, 2.0, 0.0, 4.0 * (1.0, 2.5, 0.2, 3.0, 0.1, 1.5)[k])
        res = eng.tick(2000.0 * (k + 1), arr)
        differs += [(a.kind, a.batch, a.sm_percent, a.quota_percent) for a in res.actions] != \
            [(a.kind, a.batch, a.sm_percent, a.quota_percent)
             for a in plain.tick(2000.0 * (k + 1), arr).actions]
        acts, _, _, counter = so.tick(
            {"alpha": cfg.alpha, "beta": cfg.beta, "delta": 10, "cooldown_ms": cfg.cooldown_ms,
             "r_min": cfg.r_min}, functions, otables, ocl, 2000.0 * (k + 1), 2000.0, arr,
            set(ocl.pods), kstate, {"A": 1.0, "Q": 4.0, "H": 1.0, "D": 16.0}, 1.0, last_down,
            counter, lambda pid, fid, b, s, q, g: PodInstance(pid, fid, b, s, q, g,
                                                              state=PodState.COLD_STARTING),
            lambda sm: SmPartition(sm), cold_start_ms=5000.0)
        got = [(a.function_id, a.kind.value, a.batch, a.sm_percent, a.quota_percent, pid, a.gpu_id)
               for a, pid in zip(res.actions, res.pod_ids)]
        assert got == [tuple(a) for a in acts], k
        fresh += sum(1 for a in acts if a[1] == "horizontal_up")
    assert fresh > 0
    if mult < 2.5:  # a binding SLO changes some fresh-GPU configuration
        assert differs > 0
