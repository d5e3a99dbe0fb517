"""Batched scaler tick on the B200: the drop-in for SimulationEngine._handle_scaler.

`TickEngine` uploads a scaler world — functions in sorted-id order with their perf tables,
the cluster (GPUs in sorted-id order, partition lists in insertion order, pods), Kalman
states and scale-down stamps — and runs whole ticks on the device (rapp_tick_run,
include/rapp_b200.h).  One tick reproduces, function by function in sorted order,
hs/sim.py:470-491: observed = arrivals / interval; Kalman (hs/kalman.py:45-62);
Autoscaler.scale (hs/autoscaler.py:73-234); apply (hs/sim.py:493-525: change_quota, a new
COLD_STARTING `pod-%06d` placed on its GPU, DRAINING with immediate release when idle).
The device state persists across ticks; `sync_host()` / `apply_to_host=True` keep a host
ClusterState in step when a caller needs the Python objects.
"""

from __future__ import annotations

import ctypes
import math
import sys
from typing import Mapping, Optional, Sequence

import numpy as np

from . import _lib, core
from .errors import ConfigError, FilterDegenerateError, InvariantViolation

_KIND_NAMES = ("vertical_up", "vertical_down", "horizontal_up", "horizontal_down")
_STATE_NAMES = ("cold_starting", "running", "draining")
_STATE_CODE = {name: i for i, name in enumerate(_STATE_NAMES)}
# hs/autoscaler.py:86-87 sums capability with the caller's float sum(): compensated from 3.12
SUM_MODE = 0 if sys.version_info >= (3, 12) else 1
MAX_PODS_PER_FUNCTION = 128  # kMaxPods (rapp_tick.cu); the device output block holds +4


class CallerTypes:
    """The record types of the caller's package, found from its ClusterState's module
    (hybridscale.core for the reference simulator, else this package's `core`): the
    tick emits the caller's own ActionKind / ScalingAction and creates its PodInstance /
    PodState, and applies actions to host snapshots with the caller's own allocator when
    the package has one (hs/allocator.py) — else by re-reading the device world."""

    def __init__(self, cluster):
        mod = sys.modules.get(type(cluster).__module__)
        if mod is None or not all(hasattr(mod, n) for n in
                                  ("ActionKind", "ScalingAction", "PodInstance", "PodState")):
            mod = core
        self.ActionKind = mod.ActionKind
        self.ScalingAction = mod.ScalingAction
        self.PodInstance = mod.PodInstance
        self.PodState = mod.PodState
        self.SmPartition = getattr(mod, "SmPartition", core.SmPartition)
        self.kinds = tuple(self.ActionKind(k) for k in _KIND_NAMES)
        self.states = tuple(self.PodState(k) for k in _STATE_NAMES)
        pkg = mod.__name__.rpartition(".")[0]
        alloc = sys.modules.get(pkg + ".allocator") if pkg else None
        self.allocator = alloc if alloc is not None and all(
            hasattr(alloc, n) for n in ("place_pod", "change_quota", "release_pod")) else None


class ScalerConfigC(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("beta", ctypes.c_double),
                ("cooldown_ms", ctypes.c_double), ("r_min", ctypes.c_double),
                ("delta_iq", ctypes.c_int32), ("policy", ctypes.c_int32),
                ("interval_s", ctypes.c_double), ("cold_start_ms", ctypes.c_double),
                ("kal_A", ctypes.c_double), ("kal_Q", ctypes.c_double),
                ("kal_H", ctypes.c_double), ("kal_D", ctypes.c_double),
                ("kal_P0", ctypes.c_double), ("sum_mode", ctypes.c_int32),
                ("_pad", ctypes.c_int32)]


FN_DTYPE = np.dtype([("table_id", "<i4"), ("_pad", "<i4"), ("min_rps", "<f8"),
                     ("lattice_off", "<i8"), ("lattice_len", "<i8"), ("kal_init", "<i4"),
                     ("_pad2", "<i4"), ("kal_R", "<f8"), ("kal_P", "<f8"),
                     ("last_down_ms", "<f8"), ("shape_batch", "<i4"), ("shape_sm", "<i4"),
                     ("shape_quota", "<i4"), ("_pad3", "<i4")])
POD_DTYPE = np.dtype([("fn", "<i4"), ("batch", "<i4"), ("sm", "<i4"), ("quota", "<i4"),
                      ("gpu", "<i4"), ("part", "<i4"), ("state", "<i4"), ("_pad", "<i4"),
                      ("ready_at_ms", "<f8"), ("id", "S32")])
ACTION_DTYPE = np.dtype([("fn", "<i4"), ("kind", "<i4"), ("batch", "<i4"), ("sm", "<i4"),
                         ("quota", "<i4"), ("pod", "<i4"), ("gpu", "<i4"),
                         ("released", "<i4")])
assert FN_DTYPE.itemsize == 80 and POD_DTYPE.itemsize == 72 and ACTION_DTYPE.itemsize == 32

POLICY_NAMES = ("hybrid", "horizontal-only", "exclusive-gpu")
_ALIASES = {"hybrid": "hybrid", "horizontal": "horizontal-only",
            "horizontal-only": "horizontal-only", "exclusive": "exclusive-gpu",
            "exclusive-gpu": "exclusive-gpu"}


def canonical_policy(name: str) -> str:
    """Policy name aliases of hs/policies.py:165-183; ConfigError when unknown."""
    canon = _ALIASES.get(name)
    if canon is None:
        raise ConfigError(f"unknown policy {name!r}; expected one of {POLICY_NAMES}")
    return canon


def policy_shape(policy: str, function) -> tuple[int, int, int]:
    """Fixed pod shape of the replica baselines (hs/policies.py:206-222)."""
    init = function.initial
    if policy == "exclusive-gpu":
        return init.batch, 100, 100
    return init.batch, init.sm_percent, init.quota_percent


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a.size else None


def _state_code(state) -> int:
    return _STATE_CODE[state if isinstance(state, str) else state.value]


_LOW3 = [f"{i:03d}" for i in range(1000)]


def _pod_names(c0: int, n: int) -> list[str]:
    """["pod-%06d" % c for c in range(c0, c0 + n)] (hs/sim.py:337-340), built from a table of
    the three low digits: one string concatenation per name."""
    out: list[str] = []
    c, end = c0, c0 + n
    while c < end:
        hi, lo = divmod(c, 1000)
        k = min(end - c, 1000 - lo)
        head = "pod-" + (_LOW3[hi] if hi < 1000 else str(hi))
        out.extend([head + t for t in _LOW3[lo:lo + k]])
        c += k
    return out


class TickResult:
    """One tick's output.  `raw` holds the packed action records (rapp_action) in
    emission order and `observed_rps`/`predicted_rps` the per-function rates in sorted
    function order; the reference-shaped views below are built on first access."""

    def __init__(self, engine, raw, obs, pred):
        self.raw = raw
        self.observed_rps = obs
        self.predicted_rps = pred
        self._engine = engine
        self._actions = None
        self._pod_ids = None

    @property
    def pod_ids(self) -> list[str]:
        """The pod each action refers to (new pods: their new id), in action order."""
        if self._pod_ids is None:
            pods = self.raw["pod"]
            # device pod indices are stable and the id list only grows, so the mirror read
            # at any later time gives the ids of this tick
            self._pod_ids = self._engine._ids_mirror()[pods].tolist() if len(pods) else []
        return self._pod_ids

    @property
    def actions(self) -> list:
        """The caller's ScalingAction records (horizontal_up carries pod_id None)."""
        if self._actions is None:
            # device-produced records are valid by construction: each action gets its field
            # dict directly (no frozen-dataclass __init__ / __post_init__ per action)
            e = self._engine
            fids, gids = e.fids, e.gids
            r = self.raw
            KINDS = e.types.kinds
            new, setattr_, cls = object.__new__, object.__setattr__, e.types.ScalingAction
            out = []
            app = out.append
            for f, k, b, sm, q, g, pid in zip(r["fn"].tolist(), r["kind"].tolist(),
                                               r["batch"].tolist(), r["sm"].tolist(),
                                               r["quota"].tolist(), r["gpu"].tolist(),
                                               self.pod_ids):
                a = new(cls)
                setattr_(a, "__dict__", {"function_id": fids[f], "kind": KINDS[k], "batch": b,
                                         "sm_percent": sm, "quota_percent": q,
                                         "pod_id": None if k == 2 else pid,
                                         "gpu_id": gids[g]})
                app(a)
            self._actions = out
        return self._actions

    @property
    def released(self) -> list[bool]:
        """horizontal_down of an idle pod: released at once."""
        return [bool(x) for x in self.raw["released"]]

    @property
    def observed(self) -> dict[str, float]:
        return dict(zip(self._engine.fids, self.observed_rps.tolist()))

    @property
    def predicted(self) -> dict[str, float]:
        return dict(zip(self._engine.fids, self.predicted_rps.tolist()))


class TickEngine:
    """Device-resident scaler world; `tick()` runs one _handle_scaler for all functions."""

    def __init__(self, functions: Sequence, tables: Mapping, cluster, scaler_config, *,
                 kalman_params: Optional[dict] = None, scaler_interval_ms: float = 2000.0,
                 cold_start_ms: float = 5000.0, pod_counter: int = 0,
                 kalman_states: Optional[Mapping] = None,
                 last_scale_down: Optional[Mapping[str, float]] = None,
                 promote_cold: bool = True, policy: str = "hybrid",
                 device: Optional[int] = None, slo_mask: bool = False):
        from .perf import device_table_of
        self.policy = canonical_policy(policy)
        self.cluster = cluster
        self.types = CallerTypes(cluster)
        self.config = scaler_config
        self.functions = {f.function_id: f for f in functions}
        self.fids = sorted(self.functions)
        self.fidx = {fid: i for i, fid in enumerate(self.fids)}
        kp = dict(kalman_params or {})
        kal = {"A": kp.get("A", 1.0), "Q": kp.get("Q", 4.0), "H": kp.get("H", 1.0),
               "D": kp.get("D", 16.0), "P0": kp.get("P0", 1.0)}
        self.interval_ms = float(scaler_interval_ms)
        self.cold_start_ms = float(cold_start_ms)
        # tables and batch lattices (most_efficient_config's _batch_lattice rule)
        ctx = None
        fn_arr = np.zeros(len(self.fids), dtype=FN_DTYPE)
        lattice: list[int] = []
        for i, fid in enumerate(self.fids):
            f = self.functions[fid]
            ref = f.perf_table_ref or fid
            table = tables.get(ref)
            if table is None:
                raise ConfigError(f"missing perf table {ref!r} for {fid}")
            table = device_table_of(table, device)  # any PerfTable-shaped object
            c, tid = table.device_table()
            if ctx is None:
                ctx = c
            elif c is not ctx:
                raise ConfigError("all tables of a TickEngine must share one device")
            bl = table._batch_lattice(f.allowed_batches or None)
            fn_arr[i]["table_id"] = tid
            fn_arr[i]["min_rps"] = math.nan if f.min_rps is None else float(f.min_rps)
            fn_arr[i]["lattice_off"] = len(lattice)
            fn_arr[i]["lattice_len"] = len(bl)
            lattice.extend(bl)
            st = (kalman_states or {}).get(fid)
            if st is not None:
                fn_arr[i]["kal_init"] = 1
                fn_arr[i]["kal_R"] = st.R
                fn_arr[i]["kal_P"] = st.P
            ld = (last_scale_down or {}).get(fid)
            fn_arr[i]["last_down_ms"] = -math.inf if ld is None else float(ld)
            sb, ss, sq = policy_shape(self.policy, f)
            fn_arr[i]["shape_batch"], fn_arr[i]["shape_sm"], fn_arr[i]["shape_quota"] = sb, ss, sq
        self.ctx = ctx or _lib.Context.get(device)
        # GPUs in sorted-id order; partitions in list order
        self.gids = sorted(cluster.gpus)
        self.grank = {g: i for i, g in enumerate(self.gids)}
        part_off, psm, palloc = [0], [], []
        where = {}
        for g in self.gids:
            for pos, part in enumerate(cluster.gpus[g].partitions):
                psm.append(part.sm_percent)
                palloc.append(part.quota_allocated)
                for pid in part.resident_pods:
                    where[pid] = pos
            part_off.append(len(psm))
        # pods
        self.pod_ids: list[str] = []
        self._pod_fids: list[str] = []
        self._pod_fn_pending: list[np.ndarray] = []  # function indices of new pods, unnamed
        pods = np.zeros(len(cluster.pods), dtype=POD_DTYPE)
        for i, pod in enumerate(cluster.pods.values()):
            raw = pod.pod_id.encode("utf-8")
            if len(raw) > 32 or b"\x00" in raw:
                raise ConfigError(f"pod id {pod.pod_id!r}: at most 32 UTF-8 bytes, no NUL")
            if pod.pod_id not in where:
                raise InvariantViolation(f"pod {pod.pod_id} is not resident on a partition")
            pods[i] = (self.fidx.get(pod.function_id, -1), pod.batch, pod.sm_percent,
                       pod.quota_percent, self.grank[pod.gpu_id], where[pod.pod_id],
                       _state_code(pod.state), 0,
                       float(getattr(pod, "ready_at_ms", 0.0)) if promote_cold else math.inf,
                       raw)
            self.pod_ids.append(pod.pod_id)
            self._pod_fids.append(pod.function_id)
        self.counter = int(pod_counter)
        cfg = ScalerConfigC(scaler_config.alpha, scaler_config.beta, scaler_config.cooldown_ms,
                            scaler_config.r_min, scaler_config.delta_iq,
                            0 if self.policy == "hybrid" else 1,
                            self.interval_ms / 1000.0, self.cold_start_ms, kal["A"], kal["Q"],
                            kal["H"], kal["D"], kal["P0"], SUM_MODE, 0)
        lat = np.asarray(lattice if lattice else [0], dtype=np.int64)
        po = np.asarray(part_off, dtype=np.int64)
        ps = np.asarray(psm if psm else [0], dtype=np.int32)
        pa = np.asarray(palloc if palloc else [0], dtype=np.int32)
        h = _lib.c_vp()
        _lib.check(_lib.load().rapp_tick_create(
            self.ctx.handle, ctypes.byref(cfg), len(self.fids), _ptr(fn_arr), _lib.i64ptr(lat),
            len(self.gids), _lib.i64ptr(po), _lib.i32ptr(ps), _lib.i32ptr(pa), len(pods),
            _ptr(pods), self.counter, ctypes.byref(h)), "TickEngine")
        self._h = h
        if slo_mask:
            self.set_slo({fid: self.functions[fid].slo_ms for fid in self.fids})
        # the device's own output block: kMaxPods + 4 actions per function
        self._act_buf = np.zeros(max(1, len(self.fids)) * (MAX_PODS_PER_FUNCTION + 4),
                                 dtype=ACTION_DTYPE)
        self._obs = np.zeros(max(1, len(self.fids)))
        self._pred = np.zeros(max(1, len(self.fids)))
        # the host call's persistent buffers as plain addresses (no ctypes object per tick)
        self._act_addr = self._act_buf.ctypes.data
        self._obs_addr, self._pred_addr = self._obs.ctypes.data, self._pred.ctypes.data
        self._nact = ctypes.c_int64()
        self._fids_np = np.array(self.fids, dtype=object)

    def set_slo(self, slo_ms: Optional[Mapping[str, Optional[float]]]) -> None:
        """Opt-in latency SLO for the fresh-GPU most_efficient_config of the tick
        (hs/autoscaler.py:155-165): {fid: slo in ms or None}; a configuration is feasible
        iff its throughput covers the gap AND its latency is <= the SLO (north_star (3);
        the reference never reads FunctionSpec.slo_ms, hs/core.py:96-98).  With no such
        configuration the reference's max-throughput fallback applies unchanged.  None
        restores the reference rule.  Vertical walks and covering quotas are unaffected."""
        if slo_ms is None:
            _lib.check(_lib.load().rapp_tick_set_slo(self._h, None), "set_slo")
            return
        arr = np.array([math.nan if slo_ms.get(f) is None else float(slo_ms[f])
                        for f in self.fids], dtype=np.float64)
        _lib.check(_lib.load().rapp_tick_set_slo(self._h, _ptr(arr) if len(arr) else None),
                   "set_slo")

    def close(self) -> None:
        """Frees the device world now (also done when the engine is garbage-collected)."""
        h = getattr(self, "_h", None)
        self._h = None
        if h is not None and _lib._lib is not None:
            _lib._lib.rapp_tick_destroy(h)

    def __del__(self):
        self.close()

    # -- host events between ticks ---------------------------------------------------------

    def _pod_index(self) -> dict:
        """pod id -> device pod index, extended incrementally as ticks create pods."""
        idx = getattr(self, "_index", None)
        if idx is None:
            idx = self._index = {}
        for i in range(len(idx), len(self.pod_ids)):
            idx[self.pod_ids[i]] = i
        return idx

    def release(self, pod_ids, *, apply_to_host: bool = False) -> None:
        """Pods the simulator released since the last tick (DRAINING pods whose last request
        completed, hs/sim.py:424-438), in release order."""
        ids = list(pod_ids)
        if not ids:
            return
        index = self._pod_index()
        try:
            idx = np.array([index[pid] for pid in ids], dtype=np.int64)
        except KeyError as exc:
            raise InvariantViolation(f"release of unknown pod {exc.args[0]!r}") from None
        _lib.check(_lib.load().rapp_tick_release(self._h, _lib.i64ptr(idx), len(idx)),
                   "release")
        if apply_to_host:
            alloc = self.types.allocator
            if alloc is None:
                self.sync_host()
            else:
                for pid in ids:
                    if pid in self.cluster.pods:
                        alloc.release_pod(self.cluster, pid)

    # -- one tick -----------------------------------------------------------------------

    def tick(self, now_ms: float, arrivals, idle=None, *, predicted=None,
             apply_to_host: bool = False) -> TickResult:
        """arrivals: {fid: count} or a sequence in sorted-fid order.  idle: pod ids with no
        queued / in-service work (None: every pod is idle).  predicted: {fid: rps} to skip
        the Kalman step (Autoscaler.scale semantics)."""
        lib = _lib.load()
        F = len(self.fids)
        if (type(arrivals) is np.ndarray and arrivals.dtype == np.int64
                and arrivals.flags.c_contiguous):
            arr = arrivals  # the usual host-array call: no conversion
        elif isinstance(arrivals, Mapping):
            arr = np.array([int(arrivals.get(f, 0)) for f in self.fids], dtype=np.int64)
        else:
            arr = np.ascontiguousarray(arrivals, dtype=np.int64)
        if arr.shape != (F,):
            raise ValueError(f"expected {F} arrival counts")
        if F and arr.min() < 0:
            raise ValueError("observed_rps must be non-negative")
        n = len(self.pod_ids)
        if idle is None:
            if getattr(self, "_all_idle", None) is None or len(self._all_idle) < max(1, n):
                self._all_idle = np.ones(max(1024, 2 * n), dtype=np.uint8)
                self._all_idle_addr = self._all_idle.ctypes.data
            idle_arr = self._all_idle
        else:
            idle_set = set(idle)
            idle_arr = np.fromiter((pid in idle_set for pid in self.pod_ids), dtype=np.uint8,
                                   count=n) if n else np.zeros(1, dtype=np.uint8)
        pred_in = None
        if predicted is not None:
            pred_in = np.array([float(predicted[f]) for f in self.fids], dtype=np.float64)
        nact = self._nact
        idle_addr = (self._all_idle_addr if idle_arr is getattr(self, "_all_idle", None)
                     else idle_arr.ctypes.data)
        _lib.check(lib.rapp_tick_submit(self._h, float(now_ms), arr.ctypes.data if F else None,
                                        idle_addr if idle_arr.size else None,
                                        pred_in.ctypes.data if pred_in is not None else None,
                                        len(self._act_buf)), "tick")
        try:
            self._top_up_names()  # while the tick runs on the device
        finally:  # a submitted tick is always collected (the handle accepts nothing else)
            rc = lib.rapp_tick_collect(self._h, self._act_addr, len(self._act_buf),
                                       ctypes.byref(nact), self._obs_addr, self._pred_addr)
        if rc == _lib.RAPP_E_DEGENERATE:
            raise FilterDegenerateError("H*P'*H + D == 0")
        _lib.check(rc, "tick")
        raw = self._act_buf[:nact.value].copy()
        res = self._bookkeep(raw)
        if apply_to_host:
            self._apply_host(res, float(now_ms))
        return res

    # new pod ids come from a cache of pod-%06d names for the next counter values, topped up
    # between rapp_tick_submit and rapp_tick_collect (hidden under the device tick); a tick
    # that outruns the cache names the rest itself
    _NAMES_TOPUP_MAX = 1024

    def _top_up_names(self) -> None:
        c0 = getattr(self, "_names_c0", None)
        if c0 is None:
            self._names, self._names_c0, self._names_reserve = [], self.counter, 256
            c0 = self.counter
        names = self._names
        used = self.counter - c0
        if used < 0 or used > len(names):  # counter moved outside the cache: restart it
            names.clear()
            self._names_c0 = c0 = self.counter
            used = 0
        elif used > 4096:
            del names[:used]
            self._names_c0 = c0 = self.counter
            used = 0
        short = self._names_reserve - (len(names) - used)
        if short > 0:
            names.extend(_pod_names(c0 + len(names), min(short, self._NAMES_TOPUP_MAX)))

    def _new_names(self, c0: int, k: int) -> list[str]:
        base = getattr(self, "_names_c0", None)
        if base is None:
            return _pod_names(c0, k)
        self._names_reserve = max(self._names_reserve, 2 * k)
        lo = c0 - base
        if lo < 0:
            return _pod_names(c0, k)
        have = self._names[lo:lo + k]
        if len(have) < k:
            have.extend(_pod_names(c0 + len(have), k - len(have)))
        return have

    @property
    def pod_fids(self) -> list[str]:
        """Function id of every device pod index (new pods' entries are named on demand)."""
        if self._pod_fn_pending:
            for fn in self._pod_fn_pending:
                self._pod_fids.extend(self._fids_np[fn].tolist())
            self._pod_fn_pending.clear()
        return self._pod_fids

    def _ids_mirror(self) -> np.ndarray:
        """An object-array copy of the pod id list (capacity doubling), brought up to date on
        demand, for gathering ids by device pod index."""
        ids = self.pod_ids
        mirror, n = getattr(self, "_ids_np", None), getattr(self, "_ids_n", 0)
        if mirror is None or len(mirror) < len(ids):
            grown = np.empty(max(1024, 2 * len(ids)), dtype=object)
            if mirror is not None:
                grown[:n] = mirror[:n]
            mirror = self._ids_np = grown
        if n < len(ids):
            mirror[n:len(ids)] = ids[n:]
            self._ids_n = len(ids)
        return mirror

    def _bookkeep(self, raw: np.ndarray) -> TickResult:
        """Names the pods the device created (pod-%06d in apply order, like the sim's
        counter); the per-action pod ids and the new pods' function ids are views built on
        first access (TickResult.pod_ids, TickEngine.pod_fids)."""
        pods = raw["pod"]
        ids = self.pod_ids
        new = np.flatnonzero(raw["kind"] == 2)  # horizontal_up: new pods, in order
        if len(new):
            start, c0 = len(ids), self.counter
            if not np.array_equal(pods[new], np.arange(start, start + len(new))):
                raise InvariantViolation("device pod index out of step")
            ids.extend(self._new_names(c0, len(new)))
            self._pod_fn_pending.append(raw["fn"][new])
            self.counter = c0 + len(new)
        F = len(self.fids)
        return TickResult(self, raw, self._obs[:F].copy(), self._pred[:F].copy())

    def _apply_host(self, res: TickResult, now: float) -> None:
        """Cluster effects of hs/sim.py:493-525 on the host snapshot (promotions first),
        applied by the caller's own allocator (hs/allocator.py) when its package has one,
        else re-read from the device world (`sync_host`)."""
        T = self.types
        cl = self.cluster
        cl.clock_ms = now
        alloc = T.allocator
        if alloc is None:
            self.sync_host()
            return
        cold, running, draining = T.states
        for pod in cl.pods.values():
            if pod.state.value == "cold_starting" and pod.ready_at_ms <= now:
                pod.state = running
        v_up, v_down, h_up, _ = T.kinds
        for act, pid, rel in zip(res.actions, res.pod_ids, res.released):
            if act.kind is v_up or act.kind is v_down:
                alloc.change_quota(cl, pid, act.quota_percent)
            elif act.kind is h_up:
                pod = T.PodInstance(pid, act.function_id, act.batch, act.sm_percent,
                                    act.quota_percent, act.gpu_id, state=cold,
                                    ready_at_ms=now + self.cold_start_ms)
                alloc.place_pod(cl, pod, act.gpu_id)
            else:
                cl.pods[pid].state = draining
                if rel:
                    alloc.release_pod(cl, pid)

    def sync_host(self) -> None:
        """Rewrites the host snapshot's pods and partition lists from the device world
        (pods in creation order, partitions in list order, residents in pod order)."""
        T = self.types
        cl = self.cluster
        pods = self.read_pods()
        parts = self.read_partitions()
        lists = {g: [T.SmPartition(sm, [], alloc) for sm, alloc, _ in parts[g]]
                 for g in self.gids}
        prev, fresh = cl.pods, {}
        for i, p in enumerate(pods):
            if p["state"] < 0:  # released
                continue
            pid, gid = self.pod_ids[i], self.gids[int(p["gpu"])]
            pod = prev.get(pid)
            if pod is None:  # created by a tick: COLD_STARTING until its ready time
                pod = T.PodInstance(pid, self.pod_fids[i], 0, 0, 0, gid,
                                    ready_at_ms=float(p["ready_at_ms"]))
            pod.batch, pod.sm_percent, pod.quota_percent = (int(p["batch"]), int(p["sm"]),
                                                            int(p["quota"]))
            pod.gpu_id, pod.state = gid, T.states[int(p["state"])]
            fresh[pid] = pod
            lists[gid][int(p["part"])].resident_pods.append(pid)
        prev.clear()
        prev.update(fresh)
        for g in self.gids:
            cl.gpus[g].partitions[:] = lists[g]

    # -- device state readback --------------------------------------------------------------

    def read_pods(self) -> np.ndarray:
        lib = _lib.load()
        n = ctypes.c_int64()
        _lib.check(lib.rapp_tick_read_pods(self._h, None, 0, ctypes.byref(n)))
        out = np.zeros(max(1, n.value), dtype=POD_DTYPE)
        _lib.check(lib.rapp_tick_read_pods(self._h, _ptr(out), len(out), ctypes.byref(n)))
        return out[:n.value]

    def read_partitions(self) -> dict[str, list[tuple[int, int, int]]]:
        lib = _lib.load()
        off = np.zeros(len(self.gids) + 1, dtype=np.int64)
        cap = 100 * max(1, len(self.gids))
        sm = np.zeros(cap, dtype=np.int32)
        al = np.zeros(cap, dtype=np.int32)
        npd = np.zeros(cap, dtype=np.int32)
        _lib.check(lib.rapp_tick_read_parts(self._h, _lib.i64ptr(off), _lib.i32ptr(sm),
                                            _lib.i32ptr(al), _lib.i32ptr(npd), cap))
        return {g: [(int(sm[k]), int(al[k]), int(npd[k])) for k in range(off[i], off[i + 1])]
                for i, g in enumerate(self.gids)}

    def read_functions(self) -> np.ndarray:
        out = np.zeros(max(1, len(self.fids)), dtype=FN_DTYPE)
        _lib.check(_lib.load().rapp_tick_read_fns(self._h, _ptr(out)))
        return out[:len(self.fids)]

    def device_cluster_dict(self) -> dict:
        """{gpus: [{id, partitions: [{sm, alloc, npods}]}], pods: sorted rows} — the device
        world in the same shape tests use for host snapshots (residents by count)."""
        pods = self.read_pods()
        rows = []
        for i, p in enumerate(pods):
            if p["state"] < 0:
                continue
            rows.append([self.pod_ids[i], self.pod_fids[i],
                         int(p["batch"]), int(p["sm"]), int(p["quota"]), self.gids[p["gpu"]],
                         _STATE_NAMES[int(p["state"])]])
        return {"partitions": self.read_partitions(), "pods": sorted(rows, key=str)}
