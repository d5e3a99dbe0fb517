"""ScalerConfig / Autoscaler / HybridPolicy with the reference's interface, evaluated on
the B200 (hs/autoscaler.py:28-102, hs/policies.py:25-46).

`Autoscaler.scale(function, cluster, predicted_rps)` is the single-function decision: it
uploads the snapshot as a one-function scaler world and runs the device tick with the
given rate (no Kalman step).  It does not mutate `cluster` and keeps the per-function
scale-down cooldown stamps like the reference.  For whole ticks use `tick.TickEngine`,
which decides every function in one pass with sequential-commit semantics.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Protocol

from .core import FunctionSpec, PodConfig, PodState, ScalingAction
from .errors import UnknownFunctionError, UnroutableFunctionError


@dataclass(frozen=True)
class ScalerConfig:
    alpha: float = 0.9            # scale up when R > C * alpha
    beta: float = 0.5             # scale down when R < C * beta
    delta_iq: int = 10            # quota step (percent points)
    cooldown_ms: float = 30000.0  # minimum gap between scale-downs
    r_min: float = 1.0            # never scale down at or below this rate

    def __post_init__(self):
        if not 0 < self.beta < self.alpha <= 1:
            raise ValueError(f"need 0 < beta < alpha <= 1, got alpha={self.alpha} "
                             f"beta={self.beta}")
        if not 1 <= self.delta_iq <= 100:
            raise ValueError(f"delta_iq {self.delta_iq} outside [1, 100]")
        if self.cooldown_ms < 0 or self.r_min < 0:
            raise ValueError("cooldown_ms and r_min must be non-negative")


def update_load_balancer_weights(cluster, function_id: str) -> dict[str, float]:
    """Running pods' capability shares (hs/autoscaler.py:46-55)."""
    running = [p for p in cluster.pods_of(function_id)
               if PodState(p.state.value) is PodState.RUNNING]
    if not running:
        raise UnroutableFunctionError(function_id)
    total = sum(p.capability_rps for p in running)
    if total <= 0:
        return {p.pod_id: 1.0 / len(running) for p in running}
    return {p.pod_id: p.capability_rps / total for p in running}


class Autoscaler:
    """Per-function decisions on the device; holds the scale-down cooldown stamps."""

    def __init__(self, config: ScalerConfig, tables: Mapping, *, slo_mask: bool = False):
        self.config = config
        self.tables = tables
        self.slo_mask = slo_mask  # opt-in: fresh-GPU configs must also meet function.slo_ms
        self._last_scale_down: dict[str, float] = {}

    def _table(self, function: FunctionSpec):
        table = self.tables.get(function.perf_table_ref or function.function_id)
        if table is None:
            raise UnknownFunctionError(f"no perf table for function {function.function_id}")
        return table

    def scale(self, function: FunctionSpec, cluster, predicted_rps: float
              ) -> list[ScalingAction]:
        from .tick import TickEngine
        self._table(function)
        fid = function.function_id
        # the snapshot's pod states are authoritative here (no ready-event promotion)
        eng = TickEngine([function], self.tables, cluster, self.config, promote_cold=False,
                         last_scale_down={fid: self._last_scale_down[fid]}
                         if fid in self._last_scale_down else None, slo_mask=self.slo_mask)
        res = eng.tick(cluster.clock_ms, {fid: 0}, idle=(), predicted={fid: predicted_rps})
        stamp = float(eng.read_functions()[0]["last_down_ms"])
        if stamp != float("-inf"):
            self._last_scale_down[fid] = stamp
        return res.actions


class ScalingPolicy(Protocol):
    name: str

    def initial_config(self, function: FunctionSpec) -> PodConfig:
        ...

    def decide(self, function: FunctionSpec, cluster, predicted_rps: float
               ) -> list[ScalingAction]:
        ...


class HybridPolicy:
    """The hybrid vertical/horizontal policy (hs/policies.py:36-46), B200-backed."""

    name = "hybrid"

    def __init__(self, config: ScalerConfig, tables: Mapping, *, slo_mask: bool = False):
        self._scaler = Autoscaler(config, tables, slo_mask=slo_mask)

    def initial_config(self, function: FunctionSpec) -> PodConfig:
        return function.initial

    def decide(self, function, cluster, predicted_rps):
        return self._scaler.scale(function, cluster, predicted_rps)
