"""The reference simulator with the B200 scaler tick: a `SimulationEngine` subclass.

This is the integration a `hybridscale` maintainer adds on the reference side (it lives
outside the product package: the reference is the caller).  It overrides the simulator's
per-tick hook, `SimulationEngine._handle_scaler` (hs/sim.py:470-491), with ONE device tick
(`paper_2505_01968_b200.tick.TickEngine.tick`: Kalman step, `policy.decide` and the apply
step for every function, sequential-commit semantics), then replays the returned actions —
the reference's own `ScalingAction` records — through the reference's own
`_apply_action` (hs/sim.py:493-525), so cost intervals, router resets, ready events and
quota switches happen exactly as in the reference.  Pods the simulator releases between
ticks (a DRAINING pod whose last request completes, hs/sim.py:424-438) are reported to the
device before the next tick.

    from hybridscale.sim import write_metric_csvs
    from integration.hybridscale_b200 import run
    metrics = run(trace, functions, tables, cluster, scaler_cfg, sim_cfg, "hybrid", kalman)

`tables` may hold the reference's own `PerfTable`s or the B200 `PerfTable`s: the tick uploads
either once.  Policies: the three the reference ships (`hybrid`, `horizontal-only`,
`exclusive-gpu`, by name or as the reference's policy instances); anything else raises
`ConfigError` — the device tick implements exactly those decision procedures.
"""

from __future__ import annotations

from typing import Optional

from hybridscale.core import PodState
from hybridscale.errors import ConfigError, InvariantViolation
from hybridscale.sim import SimulationEngine, TimelinePoint, _assert_monotone_curves

from paper_2505_01968_b200.tick import POLICY_NAMES, TickEngine


def _policy_settings(policy, default_config):
    """(ScalerConfig, cooldown stamps) the policy instance decides with."""
    scaler = getattr(policy, "_scaler", None)  # HybridPolicy wraps an Autoscaler
    holder = scaler if scaler is not None else policy
    return (getattr(holder, "config", None) or default_config,
            dict(getattr(holder, "_last_scale_down", {}) or {}))


class B200SimulationEngine(SimulationEngine):
    """`SimulationEngine` whose scaler ticks run on the B200 (one device tick per tick)."""

    def __init__(self, *args, device: Optional[int] = None, slo_mask: bool = False, **kwargs):
        super().__init__(*args, **kwargs)
        self._slo_mask = slo_mask  # opt-in: fresh-GPU configs also meet FunctionSpec.slo_ms
        if getattr(self.policy, "name", None) not in POLICY_NAMES:
            raise ConfigError(f"B200SimulationEngine runs the policies {POLICY_NAMES} on the "
                              f"device; got {getattr(self.policy, 'name', self.policy)!r}")
        self._device = device
        self._tick_engine: Optional[TickEngine] = None
        self._released_between_ticks: list[str] = []
        self._in_device_tick = False

    def _engine(self) -> TickEngine:
        if self._tick_engine is None:
            config, stamps = _policy_settings(self.policy, self.scaler_config)
            self._tick_engine = TickEngine(
                list(self.functions.values()), self.tables, self.cluster, config,
                kalman_params={**self._kalman_defaults, "P0": self._kalman_p0},
                scaler_interval_ms=self.cfg.scaler_interval_ms,
                cold_start_ms=self.cfg.cold_start_ms, pod_counter=self._pod_counter,
                last_scale_down=stamps, policy=self.policy.name, device=self._device,
                slo_mask=self._slo_mask)
            self._released_between_ticks.clear()  # the upload saw the current cluster
        return self._tick_engine

    def _release_pod(self, pod_id: str, now: float) -> None:
        super()._release_pod(pod_id, now)
        if not self._in_device_tick:  # the device released in-tick idle pods itself
            self._released_between_ticks.append(pod_id)

    def _handle_scaler(self, now: float) -> None:
        eng = self._engine()
        self.cluster.clock_ms = now
        if self._released_between_ticks:
            eng.release(self._released_between_ticks)
            self._released_between_ticks.clear()
        fids = eng.fids  # sorted function ids, the reference's tick order
        arrivals = [self._tick_arrivals[f] for f in fids]
        for f in fids:
            self._tick_arrivals[f] = 0
        idle = {pid for pid, rt in self._runtimes.items() if rt.idle()}
        res = eng.tick(now, arrivals, idle=idle)
        self._in_device_tick = True
        try:
            for action in res.actions:  # function order, emission order within a function
                self._apply_action(action, now)
        finally:
            self._in_device_tick = False
        if self._pod_counter != eng.counter:  # new pods are named pod-%06d in apply order
            raise InvariantViolation(f"pod counter {self._pod_counter} out of step with the "
                                     f"device tick's {eng.counter}")
        # timeline points in function order (each function's pods are final once its own
        # actions are applied; later functions never touch them)
        by_fn = {f: [] for f in fids}
        for pod in self.cluster.pods.values():
            group = by_fn.get(pod.function_id)
            if group is not None:
                group.append(pod)
        for f, obs, pred in zip(fids, res.observed_rps.tolist(), res.predicted_rps.tolist()):
            pods = by_fn[f]
            self._timeline.append(TimelinePoint(
                t_ms=now, function_id=f,
                pods=sum(1 for p in pods if p.state is not PodState.DRAINING),
                capacity_rps=sum(p.capability_rps for p in pods if p.is_running()),
                observed_rps=obs, predicted_rps=pred))
        self.cluster.validate()


def run(trace, functions, tables, cluster, scaler_config, sim_config, policy,
        kalman_params=None, *, device: Optional[int] = None, slo_mask: bool = False):
    """`hybridscale.sim.run` (hs/sim.py:623-637) with the B200 scaler tick."""
    engine = B200SimulationEngine(trace, functions, tables, cluster, scaler_config,
                                  sim_config, policy, kalman_params, device=device,
                                  slo_mask=slo_mask)
    metrics = engine.run()
    _assert_monotone_curves(metrics)
    return metrics
