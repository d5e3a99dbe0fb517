"""Scaling policies on the B200 path, name-compatible with hs/policies.py.

hybrid          vertical-first + horizontal spill (autoscaler.HybridPolicy)
horizontal-only fixed per-pod shape (function.initial), replica count only
exclusive-gpu   whole-GPU replicas (sm=100, quota=100), replica count only

Every decision is evaluated by the device tick (`tick.TickEngine`, policy code 1 for the
replica baselines: capability in pods-dict order, wanted = ceil(gap / pod_cap) fixed-shape
pods packed onto the lowest-occupancy used GPU that can take them, newest-first scale-down
of floor(excess / pod_cap) pods, cooldown shared with the hybrid policy's rules).
"""

from __future__ import annotations

from typing import Mapping

from .autoscaler import HybridPolicy, ScalerConfig, ScalingPolicy
from .core import FunctionSpec, PodConfig, ScalingAction
from .errors import UnknownFunctionError
from .tick import POLICY_NAMES, canonical_policy


class _ReplicaPolicy:
    name = "replica"

    def __init__(self, config: ScalerConfig, tables: Mapping):
        self.config = config
        self.tables = tables
        self._last_scale_down: dict[str, float] = {}

    def initial_config(self, function: FunctionSpec) -> PodConfig:
        raise NotImplementedError

    def decide(self, function: FunctionSpec, cluster, predicted_rps: float
               ) -> list[ScalingAction]:
        from .tick import TickEngine
        if self.tables.get(function.perf_table_ref or function.function_id) is None:
            raise UnknownFunctionError(f"no perf table for function {function.function_id}")
        fid = function.function_id
        eng = TickEngine([function], self.tables, cluster, self.config, promote_cold=False,
                         policy=self.name,
                         last_scale_down={fid: self._last_scale_down[fid]}
                         if fid in self._last_scale_down else None)
        res = eng.tick(cluster.clock_ms, {fid: 0}, idle=(), predicted={fid: predicted_rps})
        stamp = float(eng.read_functions()[0]["last_down_ms"])
        if stamp != float("-inf"):
            self._last_scale_down[fid] = stamp
        return res.actions


class HorizontalOnlyPolicy(_ReplicaPolicy):
    name = "horizontal-only"

    def initial_config(self, function: FunctionSpec) -> PodConfig:
        return function.initial


class ExclusiveGpuPolicy(_ReplicaPolicy):
    name = "exclusive-gpu"

    def initial_config(self, function: FunctionSpec) -> PodConfig:
        return PodConfig(batch=function.initial.batch, sm_percent=100, quota_percent=100,
                         replicas=function.initial.replicas)


def make_policy(name: str, config: ScalerConfig, tables: Mapping) -> ScalingPolicy:
    """hs/policies.py:174-183 (aliases 'horizontal', 'exclusive'; ConfigError otherwise)."""
    canon = canonical_policy(name)
    if canon == "hybrid":
        return HybridPolicy(config, tables)
    if canon == "horizontal-only":
        return HorizontalOnlyPolicy(config, tables)
    return ExclusiveGpuPolicy(config, tables)


__all__ = ["POLICY_NAMES", "ExclusiveGpuPolicy", "HorizontalOnlyPolicy", "HybridPolicy",
           "ScalingPolicy", "make_policy"]
