"""CPU oracle (test infrastructure only) for the run-metrics finalize:
SimulationEngine._finalize (hs/sim.py:586-621), _nearest_rank (:612-617) and
compute_cost (:160-175), restated over plain arrays.  Pinned against the reference's own
outputs in tests/golden/metrics.json (tests/test_metrics.py)."""

from __future__ import annotations

import math

SLO_MULTIPLIERS = [1.0 + 0.25 * i for i in range(37)]  # hs/sim.py:36


def nearest_rank(sorted_values, q):
    """hs/sim.py:612-617."""
    if not len(sorted_values):
        return float("nan")
    rank = math.ceil(q / 100.0 * len(sorted_values))
    return sorted_values[max(0, min(len(sorted_values), rank) - 1)]


def finalize(baselines, counts, latencies, intervals, price, sim_end,
             multipliers=SLO_MULTIPLIERS, pct=(50, 90, 95, 99)):
    """baselines {fid: ms}; counts {fid: (arrived, completed, rejected)}; latencies
    {fid: [ms]}; intervals [(fid, sm, quota, start, end)] in list order."""
    curve, pcts = {}, {}
    for fid in sorted(baselines):
        arrived, completed, rejected = counts[fid]
        unfinished = arrived - completed - rejected
        lat = sorted(latencies.get(fid, []))
        row = []
        for m in multipliers:
            slo = baselines[fid] * m
            late = sum(1 for x in lat if x > slo)
            bad = late + rejected + unfinished
            row.append(bad / arrived if arrived else 0.0)
        curve[fid] = row
        pcts[fid] = {f"p{q}": nearest_rank(lat, q) for q in pct}
    cost = {}
    for fid, sm, quota, start, end in intervals:  # compute_cost, hs/sim.py:160-175
        close = end if end >= 0 else sim_end
        hours = max(0.0, close - start) / 3_600_000.0
        share = (sm / 100.0) * (quota / 100.0)
        cost[fid] = cost.get(fid, 0.0) + share * hours * price
    cost = {fid: cost.get(fid, 0.0) for fid in sorted(baselines)}
    per_1k = {fid: (cost[fid] / counts[fid][1] * 1000.0 if counts[fid][1] else 0.0)
              for fid in cost}
    return curve, pcts, cost, per_1k


def finalize_np(baselines, counts, latencies, intervals, price, sim_end,
                multipliers=SLO_MULTIPLIERS, pct=(50, 90, 95, 99)):
    """The same with numpy sorting and searchsorted (exact counts) for large inputs."""
    import numpy as np
    curve, pcts = {}, {}
    for fid in sorted(baselines):
        arrived, completed, rejected = counts[fid]
        unfinished = arrived - completed - rejected
        lat = np.sort(np.asarray(latencies.get(fid, []), dtype=np.float64))
        slo = np.array([baselines[fid] * m for m in multipliers])
        late = len(lat) - np.searchsorted(lat, slo, side="right")
        curve[fid] = [(int(k) + rejected + unfinished) / arrived if arrived else 0.0
                      for k in late]
        pcts[fid] = {f"p{q}": float(nearest_rank(lat, q)) for q in pct}
    _, _, cost, per_1k = finalize({f: baselines[f] for f in baselines}, counts, {}, intervals,
                                  price, sim_end, multipliers=(), pct=())
    return curve, pcts, cost, per_1k
