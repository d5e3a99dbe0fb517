"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.  Pure-Python restatement of the reference's
scaling decision path, used to check the B200 tick kernels:

  scale()            hs/autoscaler.py:73-102 (+ _scale_up :106-166, _covering_quota
                     :168-175, _stage_new_pod :177-184, _scale_down :188-234)
  allocator queries  hs/allocator.py:17-139
  kalman_step()      hs/kalman.py:45-62
  tick()             hs/sim.py:470-491 (Kalman -> decide -> apply, per sorted function)
                     with _apply_action :493-525 reduced to its cluster effects

It works on any cluster object with the reference's attribute layout (the reference's own
ClusterState or paper_2505_01968_b200.core.ClusterState) and never imports the product.
Throughput uses the C oracle (oracle/rapp_oracle.c) for the interpolation and plain
Python IEEE division for `batch / (latency / 1000.0)`, exactly like hs/perf.py:95-98.
Pinned against the real reference by tests/test_scaler_oracle.py (golden vectors in
tests/golden/scale.json and tick.json).
"""

from __future__ import annotations

import copy
import math

from .binding import or_interp3, or_most_efficient_config

RUNNING, COLD, DRAINING = "running", "cold_starting", "draining"
V_UP, V_DOWN, H_UP, H_DOWN = "vertical_up", "vertical_down", "horizontal_up", "horizontal_down"


def _state(pod):
    s = pod.state
    return getattr(s, "value", s)


class OTable:
    """Axes + grid of one perf table (duck-typed from any PerfTable-like object)."""

    def __init__(self, table):
        self.function_id = table.function_id
        self.batches = list(table.batches)
        self.sms = list(table.sms)
        self.b = table._b_axis
        self.s = table._s_axis
        self.q = table._q_axis
        self.v = table.latency_ms

    def latency(self, b, s, q):
        if b < self.batches[0] or b > self.batches[-1]:
            raise ValueError(f"{self.function_id}: batch {b} outside table range")
        return or_interp3(self.b, self.s, self.q, self.v, float(b), float(s), float(q))

    def thr(self, b, s, q):
        return b / (self.latency(b, s, q) / 1000.0)

    def best(self, target, step, batches):
        return or_most_efficient_config(self.b, self.s, self.q, self.v, target, step, batches)


# -- allocator (hs/allocator.py) --------------------------------------------------------


def _part_of(cluster, pod):
    for part in cluster.gpus[pod.gpu_id].partitions:
        if part.sm_percent == pod.sm_percent and pod.pod_id in part.resident_pods:
            return part
    raise AssertionError(f"pod {pod.pod_id} not on a partition")


def _free_sm(gpu):
    return 100 - sum(p.sm_percent for p in gpu.partitions)


def avail_for_pod(cluster, pod):
    part = _part_of(cluster, pod)
    return pod.quota_percent + (100 - part.quota_allocated)


def best_slot(gpu):
    best, key_best = (0, 0), None
    for part in gpu.partitions:
        hr = 100 - part.quota_allocated
        if hr > 0:
            key = (part.sm_percent * hr, part.sm_percent, 1)
            if key_best is None or key > key_best:
                best, key_best = (part.sm_percent, hr), key
    free = _free_sm(gpu)
    if free > 0:
        key = (free * 100, free, 0)
        if key_best is None or key > key_best:
            best, key_best = (free, 100), key
    return best


def place(cluster, pod, gpu_id, part_factory):
    gpu = cluster.gpus[gpu_id]
    target = None
    for part in gpu.partitions:
        if part.sm_percent == pod.sm_percent and 100 - part.quota_allocated >= pod.quota_percent:
            target = part
            break
    if target is None:
        assert _free_sm(gpu) >= pod.sm_percent, "illegal placement"
        target = part_factory(pod.sm_percent)
        gpu.partitions.append(target)
    target.resident_pods.append(pod.pod_id)
    target.quota_allocated += pod.quota_percent
    pod.gpu_id = gpu_id
    cluster.pods[pod.pod_id] = pod


def set_quota(cluster, pod_id, q):
    pod = cluster.pods[pod_id]
    part = _part_of(cluster, pod)
    delta = q - pod.quota_percent
    assert 1 <= q <= 100 and part.quota_allocated + delta <= 100
    part.quota_allocated += delta
    pod.quota_percent = q


def release(cluster, pod_id):
    pod = cluster.pods[pod_id]
    gpu = cluster.gpus[pod.gpu_id]
    part = _part_of(cluster, pod)
    part.resident_pods.remove(pod_id)
    part.quota_allocated -= pod.quota_percent
    if not part.resident_pods:
        gpu.partitions.remove(part)
    del cluster.pods[pod_id]


# -- the decision (hs/autoscaler.py) ----------------------------------------------------


class Act(tuple):
    """(function_id, kind, batch, sm, quota, pod_id, gpu_id)"""


def _act(fid, kind, b, s, q, pod=None, gpu=None):
    return (fid, kind, int(b), int(s), int(q), pod, gpu)


def scale(cfg, fn, table: OTable, cluster, R, last_down, pod_factory, part_factory):
    """Returns (actions, new_last_down or None).  cfg: alpha beta delta cooldown r_min."""
    fid = fn.function_id
    now = cluster.clock_ms
    pods = sorted((p for p in cluster.pods.values() if p.function_id == fid),
                  key=lambda p: (-p.sm_percent, p.pod_id))
    pods = [p for p in pods if _state(p) != DRAINING]
    if not pods:
        return [], None
    cap = sum(table.thr(p.batch, p.sm_percent, p.quota_percent) for p in pods)
    if R > cap * cfg["alpha"]:
        return _up(cfg, fn, table, cluster, pods, R - cap * cfg["alpha"], pod_factory,
                   part_factory), None
    r_min = fn.min_rps if fn.min_rps is not None else cfg["r_min"]
    last = last_down if last_down is not None else float("-inf")
    if R < cap * cfg["beta"] and R > r_min and now - last >= cfg["cooldown_ms"]:
        acts = _down(cfg, fid, table, pods, cap - R)
        return acts, (now if acts else None)
    return [], None


class _Scratch:
    """Independent copy of the parts of a cluster a scale-up stages on (gpus with their
    partition lists, pods) — what copy.deepcopy(cluster) gives hs/autoscaler.py:111,
    without copying the unrelated function specs."""

    def __init__(self, cluster):
        self.gpus = {}
        for gid, g in cluster.gpus.items():
            ng = copy.copy(g)
            ng.partitions = []
            for p in g.partitions:
                np_ = copy.copy(p)
                np_.resident_pods = list(p.resident_pods)
                ng.partitions.append(np_)
            self.gpus[gid] = ng
        self.pods = {pid: copy.copy(p) for pid, p in cluster.pods.items()}


def _up(cfg, fn, table, cluster, pods, gap, pod_factory, part_factory):
    d = cfg["delta"]
    fid = fn.function_id
    scratch = _Scratch(cluster)
    out = []
    for pod in pods:
        if gap <= 0:
            break
        if _state(pod) != RUNNING:
            continue
        avail = avail_for_pod(scratch, scratch.pods[pod.pod_id])
        cur = table.thr(pod.batch, pod.sm_percent, pod.quota_percent)
        q, gain = pod.quota_percent, 0.0
        while q + d <= avail and gap - gain > 0:
            q += d
            gain = table.thr(pod.batch, pod.sm_percent, q) - cur
        if q > pod.quota_percent:
            set_quota(scratch, pod.pod_id, q)
            out.append(_act(fid, V_UP, pod.batch, pod.sm_percent, q, pod.pod_id, pod.gpu_id))
            gap -= gain
    bref = pods[0].batch
    if gap > 0:
        totals = {}
        for p in scratch.pods.values():  # hgo: sum(sm * quota) / 10000.0 per GPU
            totals[p.gpu_id] = totals.get(p.gpu_id, 0) + p.sm_percent * p.quota_percent
        gid = min(sorted(totals), key=lambda g: (totals[g] / 10000.0, g))
        sm, qmax = best_slot(scratch.gpus[gid])
        if sm > 0 and qmax > 0:
            if table.thr(bref, sm, qmax) > gap:
                q = qmax
                for cand in range(d, qmax + 1, d):
                    if table.thr(bref, sm, cand) >= gap:
                        q = cand
                        break
                out.append(_act(fid, H_UP, bref, sm, q, None, gid))
                place(scratch, pod_factory(f"__staged-{len(out) - 1}", fid, bref, sm, q, gid),
                      gid, part_factory)
                gap -= table.thr(bref, sm, q)
    if gap > 0:
        used = {p.gpu_id for p in scratch.pods.values()}
        free = [g for g in sorted(scratch.gpus) if g not in used]
        if free:
            b, s, q = table.best(gap, d, fn.allowed_batches or None)
            out.append(_act(fid, H_UP, b, s, q, None, free[0]))
            place(scratch, pod_factory(f"__staged-{len(out) - 1}", fid, b, s, q, free[0]),
                  free[0], part_factory)
    return out


def _down(cfg, fid, table, pods, excess):
    d = cfg["delta"]
    running = sorted((p for p in pods if _state(p) == RUNNING),
                     key=lambda p: (p.sm_percent, p.pod_id))
    alive = len(running)
    out = []
    for pod in running:
        if excess <= 0:
            break
        cur = table.thr(pod.batch, pod.sm_percent, pod.quota_percent)
        q, shed = pod.quota_percent, 0.0
        while q > 0 and excess - shed > 0:
            q = max(0, q - d)
            shed = cur if q == 0 else cur - table.thr(pod.batch, pod.sm_percent, q)
        if q == 0:
            if alive <= 1:
                floor = pod.quota_percent - d * ((pod.quota_percent - 1) // d)
                if floor < pod.quota_percent:
                    shed = cur - table.thr(pod.batch, pod.sm_percent, floor)
                    out.append(_act(fid, V_DOWN, pod.batch, pod.sm_percent, floor, pod.pod_id,
                                    pod.gpu_id))
                    excess -= shed
                continue
            alive -= 1
            out.append(_act(fid, H_DOWN, pod.batch, pod.sm_percent, 0, pod.pod_id, pod.gpu_id))
            excess -= cur
        elif q < pod.quota_percent:
            out.append(_act(fid, V_DOWN, pod.batch, pod.sm_percent, q, pod.pod_id, pod.gpu_id))
            excess -= shed
    return out


# -- replica-count baselines (hs/policies.py:49-160) -------------------------------------------


def _legal(gpu, sm, q):
    if not (1 <= sm <= 100 and 1 <= q <= 100):
        return False
    for p in gpu.partitions:
        if p.sm_percent == sm and 100 - p.quota_allocated >= q:
            return True
    return _free_sm(gpu) >= sm


def replica_decide(cfg, fn, table: OTable, cluster, R, last_down, shape, pod_factory,
                   part_factory):
    """_ReplicaPolicy.decide: returns (actions, new_last_down or None).  shape = (b, s, q)."""
    fid = fn.function_id
    sb, ss, sq = shape
    pod_cap = table.thr(sb, ss, sq)
    pods = [p for p in cluster.pods.values() if p.function_id == fid and _state(p) != DRAINING]
    if not pods:
        return [], None
    cap = sum(table.thr(p.batch, p.sm_percent, p.quota_percent) for p in pods)
    if R > cap * cfg["alpha"]:
        wanted = math.ceil((R - cap * cfg["alpha"]) / pod_cap)
        scratch = _Scratch(cluster)
        out = []
        for i in range(wanted):
            totals = {}
            for p in scratch.pods.values():
                totals[p.gpu_id] = totals.get(p.gpu_id, 0) + p.sm_percent * p.quota_percent
            cands = sorted((g for g in totals if _legal(scratch.gpus[g], ss, sq)),
                           key=lambda g: (totals[g] / 10000.0, g))
            gid = cands[0] if cands else next(
                (g for g in sorted(scratch.gpus) if g not in totals
                 and _legal(scratch.gpus[g], ss, sq)), None)
            if gid is None:
                break
            out.append(_act(fid, H_UP, sb, ss, sq, None, gid))
            place(scratch, pod_factory(f"__staged-{i}", fid, sb, ss, sq, gid), gid, part_factory)
        return out, None
    r_min = fn.min_rps if fn.min_rps is not None else cfg["r_min"]
    last = last_down if last_down is not None else float("-inf")
    if R < cap * cfg["beta"] and R > r_min and cluster.clock_ms - last >= cfg["cooldown_ms"]:
        running = sorted((p for p in pods if _state(p) == RUNNING), key=lambda p: p.pod_id,
                         reverse=True)
        removable = max(0, len(running) - 1)
        count = min(removable, int((cap - R) // pod_cap)) if pod_cap > 0 else 0
        acts = [_act(fid, H_DOWN, p.batch, p.sm_percent, 0, p.pod_id, p.gpu_id)
                for p in running[:count]]
        return acts, (cluster.clock_ms if acts else None)
    return [], None


# -- Kalman (hs/kalman.py:45-62) ------------------------------------------------------------


def kalman_step(st, observed):
    """st: dict R P A Q H D.  Returns (new dict, estimate)."""
    if observed < 0:
        raise ValueError("observed_rps must be non-negative")
    r_pred = st["A"] * st["R"]
    p_pred = st["A"] * st["P"] * st["A"] + st["Q"]
    denom = st["H"] * p_pred * st["H"] + st["D"]
    if denom == 0:
        raise ZeroDivisionError("H*P'*H + D == 0")
    gain = p_pred * st["H"] / denom
    r_new = r_pred + gain * (observed - st["H"] * r_pred)
    p_new = (1.0 - gain * st["H"]) * p_pred
    out = dict(st, R=r_new, P=p_new)
    return out, max(0.0, r_new)


# -- one scaler tick (hs/sim.py:470-491) ----------------------------------------------------


def tick(cfg, functions, tables, cluster, now, interval_ms, arrivals, idle, kstate, kdefaults,
         p0, last_down, counter, pod_factory, part_factory, cold_start_ms=5000.0,
         policy="hybrid"):
    """Mutates cluster/kstate/last_down in place.  Returns (actions with resolved pod ids,
    observed {fid: rps}, predicted {fid: rps}, new counter).  Pods whose cold start ended
    at or before `now` turn RUNNING first (ready events precede the scaler event at equal
    timestamps, hs/sim.py:40-44).  New pods get ids pod-{counter:06d} in apply order and
    start COLD_STARTING until now + cold_start_ms; a HORIZONTAL_DOWN pod is released at
    once when it is in `idle`, else marked DRAINING."""
    for pod in cluster.pods.values():
        if _state(pod) == COLD and pod.ready_at_ms <= now:
            pod.state = type(pod.state)(RUNNING)
    cluster.clock_ms = now
    interval_s = interval_ms / 1000.0
    all_actions, observed, predicted = [], {}, {}
    for fid in sorted(functions):
        fn = functions[fid]
        obs = arrivals.get(fid, 0) / interval_s
        st = kstate.get(fid)
        if st is None:
            st = dict(kdefaults, R=obs, P=p0)
        st, pred = kalman_step(st, obs)
        kstate[fid] = st
        observed[fid], predicted[fid] = obs, pred
        table = tables[fn.perf_table_ref or fid]
        if policy == "hybrid":
            acts, stamp = scale(cfg, fn, table, cluster, pred, last_down.get(fid), pod_factory,
                                part_factory)
        else:
            init = fn.initial
            shape = ((init.batch, 100, 100) if policy == "exclusive-gpu"
                     else (init.batch, init.sm_percent, init.quota_percent))
            acts, stamp = replica_decide(cfg, fn, table, cluster, pred, last_down.get(fid),
                                         shape, pod_factory, part_factory)
        if stamp is not None:
            last_down[fid] = stamp
        for a in acts:
            fid_, kind, b, s, q, pod_id, gpu_id = a
            if kind in (V_UP, V_DOWN):
                set_quota(cluster, pod_id, q)
            elif kind == H_UP:
                pod_id = f"pod-{counter:06d}"
                counter += 1
                pod = pod_factory(pod_id, fid_, b, s, q, gpu_id)
                pod.ready_at_ms = now + cold_start_ms
                place(cluster, pod, gpu_id, part_factory)
            else:
                pod = cluster.pods[pod_id]
                pod.state = type(pod.state)(DRAINING)  # the caller's PodState enum
                if pod_id in idle:
                    release(cluster, pod_id)
            all_actions.append((fid_, kind, b, s, q, pod_id, gpu_id))
    return all_actions, observed, predicted, counter


def is_nan(x):
    return isinstance(x, float) and math.isnan(x)
