"""Reference simulator experiments used for CSV parity (built through the reference's API).

Every builder takes the `hybridscale` module (the reference install: baseline/_ref on the
GPU box, the scratch copy in tests/golden/gen_golden.py) so the same inputs feed the pure
reference run and the B200 run.  Each experiment is a list of runs
(name, policy, trace, functions, tables, cluster factory, scaler, sim, kalman).
"""

from __future__ import annotations

import hashlib
import os
import random


def demo_runs(hs, config_path):
    """The reference's demo experiment (pkg/configs/demo.yaml): 2 functions, 4 GPUs, the
    step-burst scenario under all three policies — what `hybridscale run` executes
    (hs/cli.py:90-109)."""
    from hybridscale.config import load_config
    from hybridscale.sim import build_cluster
    cfg = load_config(config_path)
    runs = []
    for scenario in cfg.scenarios:
        trace = scenario.trace.build(cfg.sim.seed)
        for policy in scenario.policies:
            def cluster(cfg=cfg):
                return build_cluster(cfg.cluster.gpus, total_sm_units=cfg.cluster.total_sm_units,
                                     window_ms=cfg.sim.window_ms,
                                     price_per_hour=cfg.cluster.price_per_hour,
                                     functions=cfg.functions)
            runs.append((f"{scenario.name}-{policy}", policy, trace, cfg.functions, cfg.tables,
                         cluster, cfg.scaler, cfg.sim, cfg.kalman))
    return runs


def config3_runs(hs, horizon_ms=60000.0, policies=("hybrid",)):
    """BASELINE config 3: 100 functions with gen_tables-style surfaces (b 1..32 pow2, sm and
    quota 10..100 step 10), burst traces seeded 1000+i over a 60 s horizon, 64 GPUs, the
    demo's scaler / Kalman settings."""
    import numpy as np
    from hybridscale import (FunctionSpec, PerfTable, PodConfig, ScalerConfig, SimConfig,
                             build_cluster)
    from hybridscale.trace import merge_traces, synth_trace
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
                                  1000 + i, function_id=fid, horizon_ms=horizon_ms))
    trace = merge_traces(traces)
    scaler = ScalerConfig(alpha=0.65, beta=0.45, delta_iq=10, cooldown_ms=5000.0, r_min=1.0)
    sim = SimConfig(scaler_interval_ms=1000.0, cold_start_ms=2000.0, queue_capacity=1000,
                    seed=7, max_drain_ms=5000.0)
    kal = {"A": 1.0, "Q": 25.0, "H": 1.0, "D": 4.0, "P0": 1.0}
    return [(f"config3-{int(horizon_ms // 1000)}s-{p}", p, trace, fns, tables,
             lambda: build_cluster(64, functions=fns), scaler, sim, kal) for p in policies]


def run_to_csvs(run_fn, spec, outdir):
    """Runs one experiment with `run_fn` (hybridscale.sim.run or the B200 run) and writes
    the four metric CSVs (hs/sim.py:651-685); returns {file name: bytes}."""
    from hybridscale.sim import write_metric_csvs
    name, policy, trace, fns, tables, cluster, scaler, sim, kal = spec
    metrics = run_fn(trace, fns, tables, cluster(), scaler, sim, policy, kal)
    write_metric_csvs(metrics, outdir)
    out = {}
    for f in ("violations.csv", "latency.csv", "cost.csv", "timeline.csv"):
        with open(os.path.join(outdir, f), "rb") as fh:
            out[f] = fh.read()
    return out


def digest(files):
    return {k: {"sha256": hashlib.sha256(v).hexdigest(), "bytes": len(v)}
            for k, v in sorted(files.items())}
