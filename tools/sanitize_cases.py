"""Small workloads of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):  python tools/sanitize_cases.py CASE   (CASE in CASES)
Each case checks its result against the oracle, so a run also proves the sanitized
execution computed the right answer."""
import copy
import os
import random
import sys
import tempfile

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(os.path.join(REF, "hybridscale")):
    sys.path.append(REF)
import bench  # noqa: E402
from oracle.binding import or_interp3_many, or_most_efficient_config  # noqa: E402


def k2():
    """K2 stream interpolation (TMA ring, lane-pair cell gathers) + the literal kernel."""
    from paper_2505_01968_b200 import PerfTable, kernels
    name, b, s, q, v = bench.config2_arrays()[0]
    t = PerfTable(name, bench.BATCHES, list(range(1, 101)), list(range(1, 101)), v, device=0)
    n = 50_003  # a ragged tail past the last full TMA tile
    c = bench.gen_queries(b, s, q, n, 3, torch.device("cuda", 0))
    out = t.predict_latency_many(c).cpu().numpy()
    want = or_interp3_many(b, s, q, v, c.cpu().numpy())
    del c
    assert np.array_equal(out.view(np.int64), want.view(np.int64))
    bl = np.array([1.0, 3.0, 7.0])  # a non-uniform axis: the LUT locate
    sl = np.array([10.0, 35.0, 100.0])
    ql = np.array([5.0, 50.0, 90.0])
    vl = np.random.default_rng(1).uniform(1, 9, (3, 3, 3))
    cc = np.random.default_rng(2).uniform(0, 110, (4097, 3))
    o2 = np.empty(len(cc))
    kernels.interp3_many(bl, sl, ql, vl, cc, o2)
    assert np.array_equal(o2.view(np.int64), or_interp3_many(bl, sl, ql, vl, cc).view(np.int64))


def k3():
    """K3 lattice search (prepare, meet, min-latency, fallback, decode) incl. an SLO mask."""
    from paper_2505_01968_b200 import PerfTableSet
    tables = bench.make_config5_tables(24, seed=0, device=0)
    allowed = list(range(1, 33))
    ts = PerfTableSet([(t, allowed) for t in tables], quota_step=1)
    targets = [0.5 * bench.max_lattice_rps(t) for t in tables]
    targets[3] = 1e12  # unreachable: the fallback passes
    got = ts.search(targets)
    for t, tg, g in zip(tables, targets, got):
        assert g == or_most_efficient_config(t._b_axis, t._s_axis, t._q_axis, t.latency_ms, tg,
                                             1, allowed)
    ts.set_slo([20.0] * len(tables))
    ts.search(targets)
    _report_refs(ts)
    ts.close()


def tick():
    """The tick chain (prologue, phase A, A2, commit with its helper warps, releases, id
    formatting) over swinging-load ticks of a 60-function world, checked by the oracle."""
    from oracle import scaler_oracle as so
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    from paper_2505_01968_b200.core import PodInstance, PodState, SmPartition
    from paper_2505_01968_b200.tick import TickEngine
    fns, tables, cluster, caps = bench.make_config4_world(60, 30, seed=2, device=0)
    ocl = copy.deepcopy(cluster)
    cfg = ScalerConfig(delta_iq=10)
    eng = TickEngine(fns, tables, cluster, cfg, scaler_interval_ms=2000.0,
                     cold_start_ms=5000.0, pod_counter=len(fns))
    otables = {k: so.OTable(t) for k, t in tables.items()}
    functions = {f.function_id: f for f in fns}
    rng = random.Random(0)
    kst, ld, ctr = {}, {}, len(fns)
    for k in range(5):
        arr = bench.config4_arrivals(fns, caps, rng, 2.0, 0.0, 3.0 * (1.0, 1.5, 0.2, 2.0, 0.05)[k])
        res = eng.tick(2000.0 * (k + 1), arr)
        acts, _, _, ctr = so.tick(
            {"alpha": cfg.alpha, "beta": cfg.beta, "delta": 10, "cooldown_ms": cfg.cooldown_ms,
             "r_min": cfg.r_min}, functions, otables, ocl, 2000.0 * (k + 1), 2000.0, arr,
            set(ocl.pods), kst, {"A": 1.0, "Q": 4.0, "H": 1.0, "D": 16.0}, 1.0, ld, ctr,
            lambda pid, fid, b, s, q, g: PodInstance(pid, fid, b, s, q, g,
                                                     state=PodState.COLD_STARTING),
            lambda sm: SmPartition(sm), cold_start_ms=5000.0)
        got = [(a.function_id, a.kind.value, a.batch, a.sm_percent, a.quota_percent, pid,
                a.gpu_id) for a, pid in zip(res.actions, res.pod_ids)]
        assert got == [tuple(a) for a in acts], k
    eng.read_pods()
    del res
    _report_refs(eng)
    eng.close()


def mlp():
    """The tcgen05 MLP (stream + fused search)."""
    from paper_2505_01968_b200 import learned
    lm = learned.LearnedPerfModel.zoo(seed=0, device=0)
    c = np.random.default_rng(0).uniform([1, 1, 1], [32, 100, 100], (1000, 3))
    lat = lm.predict_many(0, c)
    ref = lm.reference_forward(0, c)
    assert np.all(np.abs(lat - ref) <= 2e-2 * ref)
    lm.search(np.array([0, 1, 2, 3]), np.array([50.0, 500.0, 5000.0, 1e9]))
    lm.close()


def ingest():
    """CSV ingest + validation kernels."""
    from paper_2505_01968_b200 import perf
    name, b, s, q, v = bench.config2_arrays()[3]
    t = perf.PerfTable(name, bench.BATCHES, list(range(1, 101)), list(range(1, 101)), v)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.csv")
        perf.save_table(t, p)
        t2 = perf.load_table(p, device=0)
        assert np.array_equal(t2.latency_ms, t.latency_ms)


def metrics():
    """Metrics finalize (violation curves, radix-select percentiles, ordered cost sums)."""
    from types import SimpleNamespace as NS
    from paper_2505_01968_b200 import metrics as m
    rng = np.random.default_rng(0)
    fids = [f"f{i}" for i in range(5)]
    lat = {f: rng.exponential(20.0, 3000).tolist() for f in fids}
    cnt = {f: NS(arrived=3010, completed=3000, rejected=4) for f in fids}
    ivs = [NS(function_id=fids[i % 5], sm_percent=20 + i, quota_percent=30, start_ms=100.0 * i,
              end_ms=100.0 * i + 777.0) for i in range(40)]
    curve, pct, cost, _ = m.finalize_arrays(fids, {f: 20.0 for f in fids}, cnt, lat, ivs, 2.48,
                                            60000.0, device=0)
    assert all(np.isfinite(cost[f]) for f in fids)


def _report_refs(obj):
    """Diagnostics: what else still references a device object at the end of its case."""
    import gc
    gc.collect()
    n = sys.getrefcount(obj) - 2
    if n > 1:
        kinds = [type(r).__name__ for r in gc.get_referrers(obj)]
        print(f"  {type(obj).__name__}: {n} references ({kinds})", flush=True)


def tick_full():
    """The benchmark-sized tick: config 4's full grid (1,000 functions, 400 GPUs, 32x91x100
    tables, quota step 1) over three swinging-load ticks, incl. the heavy scale-up tick —
    the commit's header ring, straight-line runs and staged rows at full size (hazard
    checks only: the oracle at this size is the tick GPU tests' job)."""
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    from paper_2505_01968_b200.tick import TickEngine
    fns, tables, cluster, caps = bench.make_config4_world(1000, 400, seed=0, full_grid=True,
                                                          device=0)
    eng = TickEngine(fns, tables, cluster, ScalerConfig(delta_iq=1), scaler_interval_ms=2000.0,
                     cold_start_ms=5000.0, pod_counter=len(cluster.pods))
    rng = random.Random(0)
    n = 0
    for k in range(3):
        arr = bench.config4_arrivals(fns, caps, rng, 2.0, 0.0, 3.0 * (1.0, 1.5, 0.2)[k])
        n += len(eng.tick(2000.0 * (k + 1), arr).raw)
    assert n > 500, n
    eng.read_pods()
    eng.close()


CASES = {"k2": k2, "k3": k3, "tick": tick, "mlp": mlp, "ingest": ingest, "metrics": metrics,
         "tick_full": tick_full}

if __name__ == "__main__":
    import gc
    torch.cuda.set_device(0)
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        torch.cuda.synchronize()
        print(f"{name}: ok", flush=True)
    # free every device object, then the library contexts (memcheck's leak check)
    gc.collect()
    torch.cuda.empty_cache()  # torch's caching allocator (the cases' query tensors)
    from paper_2505_01968_b200 import _lib
    _lib.Context.close_all()
