"""CPU restatement of the opt-in latency <= SLO feasibility mask (TEST INFRASTRUCTURE ONLY:
imported by tests/, never by the product).

north_star (3) asks for feasibility "latency <= SLO"; the reference's search tests only
`rps >= target` (hs/perf.py:132) and never reads FunctionSpec.slo_ms (hs/core.py:96-98), so
this is an extension with no reference behaviour to pin — parity for it is against this
restatement, built from the pinned oracle's interp3 (oracle/rapp_oracle.c):

  lattice  = _batch_lattice(batches) x table sms x range(step, 101, step)  (perf.py:119-145)
  feasible = rps >= target  and  latency <= slo_ms
  meet     = argmin (s*q, s, q, b) over feasible points
  fallback = the reference's argmin (-rps, s*q, s, q, b) over the WHOLE lattice, when no
             point is feasible (unchanged from perf.py:133-138)
"""

from __future__ import annotations

import numpy as np

from .binding import or_interp3_many, or_most_efficient_config
from .scaler_oracle import OTable


def batch_lattice(batches_axis, allowed):
    """hs/perf.py:140-145."""
    lo, hi = batches_axis[0], batches_axis[-1]
    if allowed is not None:
        inside = sorted({int(b) for b in allowed if lo <= b <= hi})
        if inside:
            return inside
    return [int(b) for b in batches_axis]


def mec_slo(b_axis, s_axis, q_axis, values, target, quota_step, batches, slo_ms):
    """most_efficient_config with the SLO mask; slo_ms None = the reference rule."""
    if slo_ms is None:
        return or_most_efficient_config(b_axis, s_axis, q_axis, values, target, quota_step,
                                        batches)
    bl = np.array(batch_lattice(list(b_axis), batches), dtype=np.float64)
    sms = np.asarray(s_axis, dtype=np.float64)
    qs = np.arange(quota_step, 101, quota_step, dtype=np.float64)
    B, S, Q = np.meshgrid(bl, sms, qs, indexing="ij")
    B, S, Q = B.ravel(), S.ravel(), Q.ravel()
    lat = or_interp3_many(b_axis, s_axis, q_axis, values, np.column_stack([B, S, Q]))
    rps = B / (lat / 1000.0)  # hs/perf.py:95-98, IEEE elementwise
    cost = S * Q
    feas = (rps >= target) & (lat <= slo_ms)
    if feas.any():
        idx = np.flatnonzero(feas)
        k = idx[np.lexsort((B[idx], Q[idx], S[idx], cost[idx]))[0]]
    else:
        k = np.lexsort((B, Q, S, cost, -rps))[0]
    return int(B[k]), int(S[k]), int(Q[k])


class OTableSLO(OTable):
    """scaler_oracle table whose most_efficient_config applies a fixed SLO (the tick's
    fresh-GPU search with TickEngine(slo_mask=True))."""

    def __init__(self, table, slo_ms):
        super().__init__(table)
        self.slo_ms = slo_ms

    def best(self, target, step, batches):
        return mec_slo(self.b, self.s, self.q, self.v, target, step, batches, self.slo_ms)
