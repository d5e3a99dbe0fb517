"""Run metrics finalize on the device: the drop-in for SimulationEngine._finalize
(hs/sim.py:586-621) and compute_cost (hs/sim.py:160-175).

`finalize(engine, sim_end)` reads the same engine state the reference method reads —
`functions`, `_counts`, `_latencies`, `_intervals`, `cfg.price_per_gpu_hour`, `_timeline` —
and returns a `RunMetrics` with the reference's fields and values (violation curve over
the 37 SLO multipliers, nearest-rank p50/p90/p95/p99, per-function cost and cost per 1k
completed requests).  A reference maintainer plugs it in by overriding `_finalize` in a
SimulationEngine subclass.  The counting, order statistics and interval
sums run in one kernel (rapp_metrics.cu); there is no CPU path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Any, Mapping, Sequence

import numpy as np

from . import _lib

SLO_MULTIPLIERS = [1.0 + 0.25 * i for i in range(37)]  # 1.00 .. 10.00 (hs/sim.py:36)
PERCENTILES = (50, 90, 95, 99)


@dataclass
class RunMetrics:
    """Field-for-field mirror of hs/sim.py:113-124."""
    multipliers: list
    violation_curve: dict
    percentiles: dict
    cost: dict
    cost_per_1k: dict
    counts: dict = field(default_factory=dict)
    timeline: Any = None
    intervals: list = field(default_factory=list)
    sim_end_ms: float = 0.0


def finalize_arrays(function_ids: Sequence[str], baselines: Mapping[str, float],
                    counts: Mapping[str, Any], latencies: Mapping[str, Sequence[float]],
                    intervals: Sequence[Any], price_per_gpu_hour: float, sim_end: float,
                    multipliers: Sequence[float] = SLO_MULTIPLIERS,
                    percentiles: Sequence[int] = PERCENTILES, *, device: int | None = None):
    """(violation_curve, percentiles, cost, cost_per_1k) dicts keyed by sorted function id.

    counts[f] has .arrived / .completed / .rejected (FunctionCounts); intervals have
    .function_id / .sm_percent / .quota_percent / .start_ms / .end_ms (PodCostInterval)."""
    fids = sorted(function_ids)
    F = len(fids)
    index = {f: i for i, f in enumerate(fids)}
    base = np.array([float(baselines[f]) for f in fids], dtype=np.float64)
    cnt = np.zeros((F, 4), dtype=np.int64)
    for i, f in enumerate(fids):
        c = counts[f]
        cnt[i] = (c.arrived, c.rejected, c.arrived - c.completed - c.rejected, c.completed)
    lens = np.array([len(latencies.get(f, ())) for f in fids], dtype=np.int64)
    lat_off = np.zeros(F + 1, dtype=np.int64)
    np.cumsum(lens, out=lat_off[1:])
    lat = np.empty(int(lat_off[-1]), dtype=np.float64)
    for i, f in enumerate(fids):
        if lens[i]:
            lat[lat_off[i]:lat_off[i + 1]] = latencies[f]
    # cost intervals grouped by function, list order kept inside each group
    own = [(index[iv.function_id], iv) for iv in intervals if iv.function_id in index]
    ivf = np.array([k for k, _ in own], dtype=np.int64)
    order = np.argsort(ivf, kind="stable")
    iv = np.array([[o.start_ms, o.end_ms, o.sm_percent, o.quota_percent] for _, o in own],
                  dtype=np.float64).reshape(-1, 4)[order]
    iv_off = np.zeros(F + 1, dtype=np.int64)
    np.cumsum(np.bincount(ivf, minlength=F)[:F], out=iv_off[1:])
    mult = np.asarray(multipliers, dtype=np.float64)
    pq = np.asarray(percentiles, dtype=np.int32)
    curve = np.empty((F, len(mult)), dtype=np.float64)
    pct = np.empty((F, len(pq)), dtype=np.float64)
    cost = np.empty(F, dtype=np.float64)
    cpk = np.empty(F, dtype=np.float64)
    ctx = _lib.Context.get(device)
    _lib.check(_lib.load().rapp_metrics_finalize(
        ctx.handle, F, _lib.dptr(base), _lib.i64ptr(cnt), _lib.i64ptr(lat_off), _lib.dptr(lat),
        _lib.i64ptr(iv_off), _lib.dptr(np.ascontiguousarray(iv)), float(price_per_gpu_hour),
        float(sim_end), len(mult), _lib.dptr(mult), len(pq), _lib.i32ptr(pq), _lib.dptr(curve),
        _lib.dptr(pct), _lib.dptr(cost), _lib.dptr(cpk)), "finalize")
    vcurve = {f: curve[i].tolist() for i, f in enumerate(fids)}
    pcts = {f: {f"p{q}": float(pct[i, j]) for j, q in enumerate(percentiles)}
            for i, f in enumerate(fids)}
    costs = {f: float(cost[i]) for i, f in enumerate(fids)}
    cost_per_1k = {f: float(cpk[i]) for i, f in enumerate(fids)}
    return vcurve, pcts, costs, cost_per_1k


def finalize(engine, sim_end: float, *, device: int | None = None) -> RunMetrics:
    """SimulationEngine._finalize (hs/sim.py:586-609) over the engine's recorded state."""
    fns = engine.functions
    vcurve, pcts, costs, cpk = finalize_arrays(
        list(fns), {f: fns[f].baseline_latency_ms for f in fns}, engine._counts,
        engine._latencies, engine._intervals, engine.cfg.price_per_gpu_hour, sim_end,
        device=device)
    return RunMetrics(multipliers=list(SLO_MULTIPLIERS), violation_curve=vcurve,
                      percentiles=pcts, cost=costs, cost_per_1k=cpk,
                      counts=dict(engine._counts), timeline=engine._timeline,
                      intervals=engine._intervals, sim_end_ms=sim_end)
