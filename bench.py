#!/usr/bin/env python3
"""Benchmark of the B200 RaPP prediction path (BASELINE.json metric, config 2 by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload stream|lattice]

Default workload (N=1 headline, BASELINE.json configs[1]): the 4-model sweep — tables
b=[1,2,4,8,16,32] x s=1..100 x q=1..100 for resnet50/vgg19/bert-base/mobilenet
(pkg/scripts/gen_tables.py:26-29 surface), 10^8 random (batch, sm%, quota%) queries per
model (1% exactly on grid nodes).  One step = interp3_many over all 4 x 10^8 queries.
  value : predictions/s with inputs resident in HBM (CUDA events, max over ranks)
  e2e   : same metric through the reference-shaped host API (kernels.interp3_many) with
          pinned host buffers: H2D of the step's queries + kernel + D2H of latencies.
Inputs (9.6 GB/GPU) are far larger than the 126 MB L2, so no flush is needed between
steps.  `--workload lattice` times config 5 instead: 3,125 functions x (32 x 100 x 100)
lattice = 1.0e9 most_efficient_config predictions per step, functions sharded over
ranks with an NCCL all-gather of the per-function (b, s, q) decisions.

Rank 0 prints ONE JSON line.  --impl reference times the reference's own compiled CPU
kernel (oracle/_ref: hs/_kernels/_grid_cy.c built from /root/reference) on all host
cores with a process pool (its nogil loop re-acquires the GIL, so threads do not scale;
SURVEY.md finding 0.6), on a bounded sample of the same workload per step.
"""

from __future__ import annotations

import argparse
import json
import os
import random
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
# the reference package (the drop-in's caller; baseline/install.sh) when installed: the B200
# path then binds its record and error types, and the tick baselines time it directly
_REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(os.path.join(_REF_INSTALL, "hybridscale")) and _REF_INSTALL not in sys.path:
    sys.path.append(_REF_INSTALL)

METRIC = "RaPP config predictions/sec and scaling decisions/tick latency at 1/2/4/8 B200"
UNIT = "predictions/s"
QUERIES_PER_MODEL = 100_000_000

# gen_tables.py:19-23 reference params; the other three are invented
MODELS = {
    "resnet50": (8.0, 1.5, 0.35, 0.65),
    "vgg19": (14.0, 4.0, 0.30, 0.70),
    "bert-base": (22.0, 5.0, 0.25, 0.75),
    "mobilenet": (3.0, 0.5, 0.50, 0.50),
}
BATCHES = [1, 2, 4, 8, 16, 32]


def surface(fixed, per_item, sm_floor, sm_weight, b, s, q):
    """pkg/scripts/gen_tables.py:26-29, evaluated left to right in float64 (vectorised)."""
    b = np.asarray(b, dtype=np.float64)[:, None, None]
    s = np.asarray(s, dtype=np.float64)[None, :, None]
    q = np.asarray(q, dtype=np.float64)[None, None, :]
    compute = fixed + per_item * b
    sm_penalty = sm_floor + sm_weight * (100.0 / s)
    return np.ascontiguousarray(compute * sm_penalty * (100.0 / q))


def config2_arrays():
    """[(name, b_axis, s_axis, q_axis, values)] for the 4-model sweep."""
    s = list(range(1, 101))
    q = list(range(1, 101))
    out = []
    for name, p in MODELS.items():
        out.append((name, np.array(BATCHES, float), np.array(s, float), np.array(q, float),
                    surface(*p, BATCHES, s, q)))
    return out


def make_config5_tables(n, seed=0, device=None, upload=True):
    """Config 5 tables: b=[1..32 pow2] x s=1..100 x q=10..100/10 per function, random
    gen_tables parameters (fixed~U(4,20), per_item~U(0.5,4),
    sm_floor~U(0.2,0.4)).  The lattice a search walks is B x table.sms x quota steps
    (hs/perf.py:123-125), so the sm axis is 1..100 to give the 32x100x100 lattice."""
    from paper_2505_01968_b200 import PerfTable
    rng = random.Random(seed)
    s = list(range(1, 101))
    q = list(range(10, 101, 10))
    tables = []
    for i in range(n):
        fixed, per, floor = rng.uniform(4, 20), rng.uniform(0.5, 4), rng.uniform(0.2, 0.4)
        tables.append(PerfTable(f"fn-{i:05d}", BATCHES, s, q,
                                surface(fixed, per, floor, 1.0 - floor, BATCHES, s, q),
                                device=device) if upload else
                      _HostTable(BATCHES, s, q,
                                 surface(fixed, per, floor, 1.0 - floor, BATCHES, s, q)))
    return tables


class _HostTable:
    """Axes + grid only (CPU-baseline workers never touch the device)."""

    def __init__(self, b, s, q, lat):
        self.batches = list(b)
        self._b_axis, self._s_axis, self._q_axis = (np.asarray(a, dtype=np.float64)
                                                    for a in (b, s, q))
        self.latency_ms = lat


def make_config4_world(nfn=1000, ngpu=400, seed=0, full_grid=False, device=None):
    """Config 4: nfn functions with random gen_tables surfaces (6x10x10:
    b=1..32 pow2, s,q=10..100 step 10; full_grid: 32x91x100 and delta 1), one pod each at
    (b=8, s=20, q=20) placed round-robin over ngpu GPUs.  Returns (functions, tables,
    cluster, caps) with caps[f] = throughput of the initial pod."""
    from paper_2505_01968_b200 import PerfTable
    from paper_2505_01968_b200.core import (ClusterState, FunctionSpec, GpuDevice, PodConfig,
                                            PodInstance, PodState)
    rng = random.Random(seed)
    if full_grid:
        bs, ss, qs = list(range(1, 33)), list(range(10, 101)), list(range(1, 101))
    else:
        bs, ss, qs = BATCHES, list(range(10, 101, 10)), list(range(10, 101, 10))
    fns, tables, caps = [], {}, {}
    for i in range(nfn):
        fid = f"fn-{i:04d}"
        fixed, per, floor = rng.uniform(4, 20), rng.uniform(0.5, 4), rng.uniform(0.2, 0.4)
        lat = surface(fixed, per, floor, 1.0 - floor, bs, ss, qs)
        tables[fid] = PerfTable(fid, bs, ss, qs, lat, device=device)
        fns.append(FunctionSpec(function_id=fid, baseline_latency_ms=20.0, perf_table_ref=fid,
                                allowed_batches=list(BATCHES), initial=PodConfig(8, 20, 20)))
        node = lat[bs.index(8), ss.index(20), qs.index(20)]
        caps[fid] = 8 / (node / 1000.0)
    cluster = ClusterState(gpus={f"gpu-{g:03d}": GpuDevice(f"gpu-{g:03d}") for g in range(ngpu)},
                           functions={f.function_id: f for f in fns})
    for i, f in enumerate(fns):
        pod = PodInstance(f"pod-{i:06d}", f.function_id, 8, 20, 20, "",
                          state=PodState.RUNNING)
        place_initial(cluster, pod, f"gpu-{i % ngpu:03d}")
    return fns, tables, cluster, caps


def place_initial(cluster, pod, gpu_id):
    """World construction: the pod joins the GPU's first same-sm partition with quota room
    for it, else opens a new partition (the placement rule of hs/allocator.py:55-108; the
    bench's initial worlds never exceed a GPU's SM share)."""
    from paper_2505_01968_b200.core import SmPartition
    parts = cluster.gpus[gpu_id].partitions
    part = next((p for p in parts if p.sm_percent == pod.sm_percent
                 and p.quota_allocated + pod.quota_percent <= 100), None)
    if part is None:
        part = SmPartition(pod.sm_percent)
        parts.append(part)
    part.resident_pods.append(pod.pod_id)
    part.quota_allocated += pod.quota_percent
    pod.gpu_id = gpu_id
    cluster.pods[pod.pod_id] = pod


def config4_arrivals(fns, caps, rng, interval_s, lo=0.0, hi=3.0):
    """Per-tick request counts giving observed rates ~ U(lo, hi) x initial capability."""
    return {f.function_id: int(rng.uniform(lo, hi) * caps[f.function_id] * interval_s)
            for f in fns}


def max_lattice_rps(table):
    """Max throughput of the (monotone) table's lattice: the (b_max, s_max, q=100) node."""
    lat = float(table.latency_ms[-1, -1, -1])
    return table.batches[-1] / (lat / 1000.0)


def load_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.6)  # let the sampler start before the timed region
        except Exception:
            self.proc = None
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        import datetime
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            # keep samples inside the timed region (with 50 ms slack either side)
            if ts is not None and self.t0 is not None and self.t1 is not None and \
                    not (self.t0 - 0.05 <= ts <= self.t1 + 0.05):
                continue
            try:
                sms.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sms:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sms)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


# ----------------------------------------------------------------------------------------
# distributed plumbing
# ----------------------------------------------------------------------------------------


_ALL_CPUS = None  # the process's CPU set before numa_bind (the CPU baselines use all of it)


class all_cpus:
    """Context: the whole host CPU set (CPU-baseline process pools inherit it)."""

    def __enter__(self):
        self.saved = os.sched_getaffinity(0)
        if _ALL_CPUS:
            os.sched_setaffinity(0, _ALL_CPUS)

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.saved)


def numa_bind(local):
    """Best effort: run this rank's host threads on the CPUs of its GPU's NUMA node, so the
    pinned staging buffers allocated afterwards are local to the GPU's PCIe root (the e2e
    copies are PCIe-bound).  No-op when the topology is not exposed."""
    import torch
    try:
        pr = torch.cuda.get_device_properties(local)
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as fh:
            node = int(fh.read().strip())
        if node < 0:
            return None
        with open(f"/sys/devices/system/node/node{node}/cpulist") as fh:
            cpus = set()
            for part in fh.read().strip().split(","):
                lo, _, hi = part.partition("-")
                cpus.update(range(int(lo), int(hi or lo) + 1))
        if cpus:
            global _ALL_CPUS
            _ALL_CPUS = os.sched_getaffinity(0)
            os.sched_setaffinity(0, cpus)
            return node
    except (OSError, ValueError, AttributeError):
        pass
    return None


def dist_init(gpus):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        if rank == 0:  # NCCL's init log (nRanks, transport) from rank 0 only, before its line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    numa_bind(local)
    return rank, world, local


def barrier(world):
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(x, world):
    import torch
    import torch.distributed as dist
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------------------
# our arm: stream workload (config 2)
# ----------------------------------------------------------------------------------------


def gen_queries(b, s, q, n, seed, device):
    """Uniform over the axis ranges, 1% of rows exactly on grid nodes (device RNG)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    c = torch.empty((n, 3), dtype=torch.float64, device=device)
    for col, axis in enumerate((b, s, q)):
        lo, hi = float(axis[0]), float(axis[-1])
        c[:, col].uniform_(lo, hi, generator=g)
    m = n // 100
    ax = [torch.from_numpy(a).to(device) for a in (b, s, q)]
    for col in range(3):
        idx = torch.randint(0, len(ax[col]), (m,), generator=g, device=device)
        c[:m, col] = ax[col][idx]
    return c


def transfer_ceiling(h_in, h_out, dev, reps=3):
    """Queries/s the PCIe link sustains for the e2e stream's copies alone: h_in (n, 3)
    float64 host->device and h_out (n,) float64 device->host, pinned, on two streams."""
    import torch
    d_in = torch.empty(h_in.shape, dtype=h_in.dtype, device=dev)
    d_out = torch.empty(h_out.shape, dtype=h_out.dtype, device=dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best = float("inf")
    for _ in range(reps + 1):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        with torch.cuda.stream(s_in):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s_out):
            h_out.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize(dev)
        best = min(best, time.perf_counter() - t0)
    del d_in, d_out
    return h_in.shape[0] / best


def run_stream(args, rank, world, local):
    import torch
    from paper_2505_01968_b200 import PerfTable, _lib, kernels
    dev = torch.device("cuda", local)
    n = args.queries
    tables, coords, outs = [], [], []
    for mi, (name, b, s, q, v) in enumerate(config2_arrays()):
        t = PerfTable(name, BATCHES, list(range(1, 101)), list(range(1, 101)), v, device=local)
        t.device_table()
        tables.append(t)
        coords.append(gen_queries(b, s, q, n, 1000 * rank + mi, dev))
        outs.append(torch.empty(n, dtype=torch.float64, device=dev))
    stream = torch.cuda.current_stream(dev)
    preds_per_step = len(tables) * n

    def step(evs=None):
        for k, t in enumerate(tables):
            if evs is not None:
                evs[k][0].record(stream)
            t.predict_latency_many(coords[k], outs[k], stream=stream.cuda_stream)
            if evs is not None:
                evs[k][1].record(stream)

    for _ in range(args.warmup):
        step()
    barrier(world)
    launches0 = _lib.launch_count()
    kev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in tables] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        clk.mark_start()
        start.record(stream)
        for i in range(args.steps):
            step(kev[i])
        end.record(stream)
        torch.cuda.synchronize()
        clk.mark_end()
    launches = _lib.launch_count() - launches0
    barrier(world)
    ms = max_over_ranks(start.elapsed_time(end), world)
    kernel_ms = [a.elapsed_time(b) for row in kev for (a, b) in row]
    avg_launch_ms = float(np.mean(kernel_ms))
    value = world * preds_per_step * args.steps / (ms / 1000.0)

    # e2e: the reference-shaped host API with pinned host buffers, copies inside the timing
    e2e = None
    if not args.no_e2e:
        # each e2e step streams 2.5e7 queries per model (1e8 predictions, 2.4 GB in) from
        # pinned host memory — a bounded slice of the same workload, same metric
        ne = min(n, 25_000_000)
        hc = [c[:ne].cpu().pin_memory() for c in coords]
        ho = [torch.empty(ne, dtype=torch.float64).pin_memory() for _ in tables]
        arrays = config2_arrays()

        def e2e_step():
            for k, (_, b, s, q, v) in enumerate(arrays):
                kernels.interp3_many(b, s, q, v, hc[k].numpy(), ho[k].numpy())

        e2e_step()
        ok = all(np.array_equal(ho[k].numpy().view(np.int64),
                                outs[k][:ne].cpu().numpy().view(np.int64))
                 for k in range(len(ho)))
        if not ok:
            raise RuntimeError("e2e host path disagrees with the device path")
        barrier(world)
        e2e_steps = max(1, min(args.steps, 10))
        e2e_preds = len(tables) * ne
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, world)
        e2e = {"value": world * e2e_preds * e2e_steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": e2e_preds * 24, "d2h_bytes_per_step": e2e_preds * 8,
               "steps": e2e_steps, "api": "kernels.interp3_many, pinned host buffers"}
        # the link's own ceiling for this traffic: the same bytes moved by bare copies
        # (24 B/query in and 8 B/query out on two streams, both directions at once)
        link = transfer_ceiling(hc[0], ho[0], dev)
        e2e["link"] = {"preds_per_s": round(world * link, 1), "unit": UNIT,
                       "frac": round(e2e["value"] / (world * link), 4),
                       "what": "cudaMemcpyAsync H2D 24 B + D2H 8 B per query, pinned, "
                               "concurrent on two streams (no kernel)"}

    peak, peak_kind = load_peak()
    alg_bytes = 32.0 * n  # 24 B coords read + 8 B latency written per prediction
    achieved = alg_bytes / (avg_launch_ms / 1000.0) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": load_traffic(n),
                "kernel": "k_interp_fast", "peak_source": peak_kind, "alg_B_per_pred": 32}
    cfg = {"workload": "config2: 4 models x 1e8 random queries/GPU, tables 6x100x100",
           "queries_per_step_per_gpu": preds_per_step, "l2": "inputs 9.6 GB/GPU >> L2",
           "parallelism": f"replicas x{world} (no collective on the data path)"}
    return {"value": value, "ms": ms, "roofline": roofline, "e2e": e2e, "config": cfg,
            "launches": launches, "clocks": clk.summary(), "dtype": "f64",
            "scaling": "weak", "avg_launch_ms": avg_launch_ms}


def load_traffic(n, kernel="k_interp_stream", field="dram_bytes_per_prediction"):
    """DRAM bytes per launch of a kernel from the committed ncu capture (per-unit figure x
    the units one launch processes)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            per_unit = float(json.load(fh)[kernel][field])
        return round(per_unit * n)
    except Exception:
        return None


# ----------------------------------------------------------------------------------------
# our arm: lattice workload (config 5)
# ----------------------------------------------------------------------------------------


def lattice_fp64_ops(table, batches, step):
    """FP64 operations K3 executes per lattice point of one function (algorithmic work of
    the run formulation, rapp_search.cu): the lattice's sm values are table nodes, so a
    row value is one quota lerp (sub/mul/add); batch entries are grouped in runs by their
    lower row (node hits and clamps join the run at their row), each run needs its lower
    row (3 ops), its upper row unless the run above produced it (3 ops) and one sub; every
    point is the final batch lerp (mul, add) plus the feasibility compare."""
    ax = list(table._b_axis)
    last = len(ax) - 1
    runs = []
    for b in batches:
        if b <= ax[0]:
            lo = 0
        elif b >= ax[-1]:
            lo = last
        else:
            lo = max(i for i in range(len(ax)) if ax[i] <= b)
        if not runs or runs[-1] != lo:
            runs.append(lo)
    per_pair, up = 3 * len(batches), -2
    for lo in reversed(runs):
        per_pair += 3
        if lo != last:
            per_pair += 1 + (0 if lo + 1 == up else 3)
        up = lo
    return per_pair / len(batches)


def fp64_peak(local):
    """Measured non-FMA FP64 instruction rate (ops/s) of this device (rapp_probe_fp64)."""
    import ctypes
    from paper_2505_01968_b200 import _lib
    a, m = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.load().rapp_probe_fp64(int(local), ctypes.byref(a), ctypes.byref(m)))
    return min(a.value, m.value)


def run_lattice(args, rank, world, local):
    import ctypes
    import torch
    from paper_2505_01968_b200 import PerfTableSet, _lib
    dev = torch.device("cuda", local)
    nfn = args.functions
    tables = make_config5_tables(nfn, seed=0, device=local)
    allowed = list(range(1, 33))
    from paper_2505_01968_b200.shard import search_sharded, shard_range
    tset = PerfTableSet([(t, allowed) for t in tables], quota_step=1)
    host_targets = np.array([0.5 * max_lattice_rps(t) for t in tables], dtype=np.float64)
    targets = torch.from_numpy(host_targets).to(dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        # functions sharded over ranks; one NCCL all-gather of the (b, s, q) decisions
        return search_sharded(tset, targets, rank, world, stream=stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    barrier(world)
    lib = _lib.load()
    _lib.check(lib.rapp_mec_plan_timing(tset._plan, 1))
    launches0 = _lib.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        clk.mark_start()
        start.record(stream)
        for _ in range(args.steps):
            step()
        end.record(stream)
        torch.cuda.synchronize()
        clk.mark_end()
    launches = _lib.launch_count() - launches0
    k_ms, k_n = ctypes.c_double(), ctypes.c_int64()
    _lib.check(lib.rapp_mec_plan_kernel_time(tset._plan, ctypes.byref(k_ms), ctypes.byref(k_n)))
    _lib.check(lib.rapp_mec_plan_timing(tset._plan, 0))
    barrier(world)
    ms = max_over_ranks(start.elapsed_time(end), world)
    points = tset.points
    value = points * args.steps / (ms / 1000.0)
    # roofline of the dominant kernel (the K3 meet pass) against the measured FP64 rate
    f0, f1 = shard_range(nfn, rank, world)
    my_points = points * (f1 - f0) / nfn
    ops_pt = lattice_fp64_ops(tables[0], allowed, 1)
    kern_s = k_ms.value / 1000.0 / max(1, k_n.value)
    achieved = my_points * ops_pt / kern_s / 1e12
    peak = fp64_peak(local) / 1e12
    roof = {"bound": "fp64", "achieved": round(achieved, 3), "peak": round(peak, 3),
            "unit": "Tops/s", "frac": round(achieved / peak, 4),
            "traffic": load_traffic(my_points, "k_mec_lattice", "dram_bytes_per_point"),
            "kernel": "k_mec_lattice<meet> (rapp_search.cu)",
            "peak_source": "measured: rapp_probe_fp64 (independent __dadd_rn/__dmul_rn chains "
                           "on every SM, min of the two rates)",
            "fp64_ops_per_point": round(ops_pt, 4),
            "naive_fp64_ops_per_point": 30.30,
            "kernel_ms_per_launch": round(kern_s * 1000.0, 4),
            "kernel_share_of_step": round(k_ms.value / max(1e-9, start.elapsed_time(end)), 4),
            "note": "the kernel is issue-bound (integer/select work beside the FP64 ops); "
                    "HBM traffic is the tables once (48 KB/function)"}
    # end to end through the public API: host targets -> H2D, search, D2H decisions
    e2e = None
    if not args.no_e2e:
        pinned = torch.from_numpy(host_targets).pin_memory()
        out_host = torch.empty((nfn, 3), dtype=torch.int32).pin_memory()
        d_t = torch.empty_like(targets)

        def e2e_step():
            d_t.copy_(pinned, non_blocking=True)
            res = search_sharded(tset, d_t, rank, world, stream=stream.cuda_stream)
            out_host.copy_(res, non_blocking=True)
        for _ in range(2):
            e2e_step()
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nrep = max(3, args.steps // 2)
        for _ in range(nrep):
            e2e_step()
        torch.cuda.synchronize()
        dt = max_over_ranks((time.perf_counter() - t0) * 1000.0, world)
        e2e = {"value": points * nrep / (dt / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": nfn * 8, "d2h_bytes_per_step": nfn * 12, "steps": nrep,
               "api": "shard.search_sharded over PerfTableSet (C ABI rapp_mec_plan_run_dev), "
                      "pinned host targets in, (b, s, q) decisions out"}
    cfg = {"workload": f"config5: {nfn} functions x 32 batches x 100 sm x 100 quota lattice "
           "(most_efficient_config, target 0.5 x max rps), tables 6x100x10",
           "points_per_step": points, "parallelism": f"functions sharded x{world}, NCCL "
           "all-gather of decisions",
           "l2": "tables 150 MB > 126 MB L2, each read once per step (no flush needed)"}
    return {"value": value, "ms": ms, "roofline": roof, "e2e": e2e, "config": cfg,
            "launches": launches, "clocks": clk.summary(), "dtype": "f64",
            "scaling": "strong"}


def run_mlp(args, rank, world, local, n_per_model=None):
    """Learned RaPP predictor (§8(f) row 4, parity unpinned): the fused feature-assembly +
    tcgen05 MLP over config-2-shaped query streams of the 4 zoo models.  Roofline: tensor
    FLOPs per prediction = 2 * (64*128 + 128*128 + 128) = 49,408 against the measured bf16
    peak."""
    import torch
    from paper_2505_01968_b200 import _lib, learned
    dev = torch.device("cuda", local)
    n = n_per_model or min(args.queries, 50_000_000)
    lm = learned.LearnedPerfModel.zoo(seed=0, device=local)
    coords, outs = [], []
    for mi, (_, b, s, q, _v) in enumerate(config2_arrays()):
        coords.append(gen_queries(b, s, q, n, 77 + 1000 * rank + mi, dev))
        outs.append(torch.empty(n, dtype=torch.float64, device=dev))
    stream = torch.cuda.current_stream(dev)
    steps = max(3, args.steps // 10)

    def step(evs=None):
        for k in range(len(coords)):
            if evs is not None:
                evs[k][0].record(stream)
            lm.predict_many_dev(k, coords[k], outs[k], stream=stream.cuda_stream)
            if evs is not None:
                evs[k][1].record(stream)

    for _ in range(args.warmup):
        step()
    barrier(world)
    launches0 = _lib.launch_count()
    kev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in coords] for _ in range(steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        clk.mark_start()
        start.record(stream)
        for i in range(steps):
            step(kev[i])
        end.record(stream)
        torch.cuda.synchronize()
        clk.mark_end()
    launches = _lib.launch_count() - launches0
    ms = max_over_ranks(start.elapsed_time(end), world)
    per_launch = float(np.mean([a.elapsed_time(b) for row in kev for (a, b) in row]))
    value = world * len(coords) * n * steps / (ms / 1000.0)
    flops = 2.0 * (64 * 128 + 128 * 128 + 128)  # layer 3 runs as an N=16 MMA (53,248 issued)
    achieved = flops * n / (per_launch / 1000.0) / 1e12
    peak = load_bf16_peak()
    roof = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": load_traffic(n, "k_mlp_stream"),
            "kernel": "k_mlp_stream (rapp_mlp.cu, tcgen05.mma kind::f16 M128 N128 K16)",
            "flops_per_prediction": flops, "hbm_bytes_per_prediction": 32,
            "achieved_hbm_gbs": round(32.0 * n / (per_launch / 1000.0) / 1e9, 1)}
    # e2e through the host API (pageable numpy in and out)
    e2e = None
    if not args.no_e2e:
        ne = 25_000_000
        hc = coords[0][:ne].cpu().pin_memory()
        ho = torch.empty(ne, dtype=torch.float64).pin_memory()
        lm.predict_many(0, hc.numpy(), ho.numpy())
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 3
        for _ in range(reps):
            lm.predict_many(0, hc.numpy(), ho.numpy())
        dt = time.perf_counter() - t0
        e2e = {"value": ne * reps / dt, "unit": UNIT, "h2d_bytes_per_step": ne * 24,
               "d2h_bytes_per_step": ne * 8, "steps": reps,
               "api": "learned.LearnedPerfModel.predict_many (C ABI rapp_mlp_predict_host, "
                      "pinned host buffers)"}
    # CPU baseline: the same forward (fp32, torch on the host cores) on a bounded sample
    import torch as _t
    sample = coords[0][:200_000].cpu().numpy()
    threads = _t.get_num_threads()
    with all_cpus():
        t0 = time.perf_counter()
        lm.reference_forward(0, sample)
        cdt = time.perf_counter() - t0
    cpu = {"value": len(sample) / cdt, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"{len(sample)} queries through the fp32 torch forward on the host"}
    # the fused search over the learned predictions (feasibility + packed-key argmin in
    # the layer-2 epilogue): config-5-shaped lattices, 32 batches x 100 sm x 100 quota
    nfs = 625
    bl = torch.arange(1, 33, dtype=torch.float64, device=dev)
    sl = torch.arange(1, 101, dtype=torch.float64, device=dev)
    mof = torch.arange(nfs, dtype=torch.int32, device=dev) % len(lm.names)
    tg = torch.full((nfs,), 2000.0, dtype=torch.float64, device=dev)
    lm.search_dev(mof, tg, bl, sl, 1)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(3):
        lm.search_dev(mof, tg, bl, sl, 1, stream=stream.cuda_stream)
    s1.record(stream)
    torch.cuda.synchronize()
    search = {"points_per_s": nfs * 32 * 100 * 100 * 3 / (s0.elapsed_time(s1) / 1000.0),
              "functions": nfs, "lattice": "32 batches x 100 sm x 100 quota",
              "ms_per_search": s0.elapsed_time(s1) / 3,
              "api": "LearnedPerfModel.search_dev (rapp_mlp_search_dev)"}
    cfg = {"workload": "learned RaPP MLP (zoo: resnet50, vgg19, bert-base, mobilenet; "
           "64 features -> 128 -> 128 -> 1, random weights), config-2-shaped query streams",
           "queries_per_step": len(coords) * n, "parity": "unpinned (no reference model); "
           "checked against a torch fp32 forward, rel tol 2e-2"}
    return {"value": value, "ms": ms, "steps": steps, "roofline": roof, "e2e": e2e,
            "cpu_baseline": cpu, "config": cfg, "launches": launches, "clocks": clk.summary(),
            "dtype": "bf16", "scaling": "weak", "search": search}


def load_bf16_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["bf16_tflops"])
    except Exception:
        return 2250.0


_LW = {}


def _lattice_worker_init(nfn_sample):
    from oracle.binding import load_oracle
    load_oracle()
    tables = make_config5_tables(nfn_sample, seed=0, device=None, upload=False)
    _LW["work"] = [(t, 0.5 * max_lattice_rps(t)) for t in tables]


def _lattice_worker_run(_):
    from oracle.binding import or_most_efficient_config
    for t, target in _LW["work"]:
        or_most_efficient_config(t._b_axis, t._s_axis, t._q_axis, t.latency_ms, target, 1,
                                 list(range(1, 33)))
    return len(_LW["work"])


def lattice_cpu_baseline_all():
    with all_cpus():
        return lattice_cpu_baseline()


def lattice_cpu_baseline(fn_per_proc=25, steps=3, procs=None):
    """The C restatement of most_efficient_config (oracle/rapp_oracle.c; the reference's
    search is Python, hs/perf.py:104-145, and cannot travel to the GPU box) over a process
    pool: config-5 lattices per second of host time."""
    import multiprocessing as mp
    procs = procs or host_cores()
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs, initializer=_lattice_worker_init, initargs=(fn_per_proc,)) as pool:
        pool.map(_lattice_worker_run, range(procs))
        t0 = time.perf_counter()
        for _ in range(steps):
            pool.map(_lattice_worker_run, range(procs))
        dt = time.perf_counter() - t0
    pts = steps * procs * fn_per_proc * 32 * 100 * 100
    return {"value": pts / dt, "unit": UNIT, "cores": procs, "kind": "port",
            "sample": f"{fn_per_proc} config-5 functions (32x100x100 lattice each) per process "
                      f"per step, {procs} processes, {steps} steps ({pts} points, {dt:.2f} s)"}


# ----------------------------------------------------------------------------------------
# tick workload (config 4): whole scaler ticks for 1,000 functions on 400 simulated GPUs
# ----------------------------------------------------------------------------------------


def run_tick(args, local, ticks=None, warmup=None, full_grid=False, nfn=1000, ngpu=400):
    """Device µs per tick (CUDA events around rapp_tick_run_dev, inputs resident) and
    end-to-end µs per tick through TickEngine.tick (H2D arrivals + idle flags, kernels,
    D2H of the ordered action list and rates).  Config 4: nfn=1000, ngpu=400; the
    config-3 tick size is nfn=100, ngpu=64."""
    import ctypes
    import torch
    from paper_2505_01968_b200 import _lib
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    from paper_2505_01968_b200.tick import TickEngine
    ticks = ticks or args.ticks
    warmup = warmup if warmup is not None else 3
    dev = torch.device("cuda", local)
    fns, tables, cluster, caps = make_config4_world(nfn, ngpu, seed=0, full_grid=full_grid,
                                                    device=local)
    cfg = ScalerConfig(delta_iq=1 if full_grid else 10)
    interval_ms = 2000.0
    rng = random.Random(0)

    def arrivals_for(k):
        swing = (1.0, 1.5, 0.2, 2.0, 0.05)[k % 5]
        a = config4_arrivals(fns, caps, rng, interval_ms / 1000.0, 0.0, 3.0 * swing)
        return np.array([a[f.function_id] for f in sorted(fns, key=lambda f: f.function_id)],
                        dtype=np.int64)

    import copy
    cluster0 = copy.deepcopy(cluster)
    t0 = time.perf_counter()
    eng = TickEngine(fns, tables, cluster, cfg, scaler_interval_ms=interval_ms,
                     cold_start_ms=5000.0, pod_counter=len(cluster.pods), device=local)
    build_s = time.perf_counter() - t0
    lib = _lib.load()
    stream = torch.cuda.current_stream(dev)
    total = warmup + ticks
    d_arr = [torch.from_numpy(arrivals_for(k)).to(dev) for k in range(total)]
    d_idle = torch.ones(1 << 20, dtype=torch.uint8, device=dev)
    pa, pc = _lib.c_vp(), _lib.c_vp()
    _lib.check(lib.rapp_tick_outputs_dev(eng._h, ctypes.byref(pa), ctypes.byref(pc), None, None))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(total)]
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        clk.mark_start()
        for k in range(total):
            evs[k][0].record(stream)
            _lib.check(lib.rapp_tick_run_dev(eng._h, interval_ms * (k + 1),
                                             d_arr[k].data_ptr(), d_idle.data_ptr(),
                                             stream.cuda_stream))
            evs[k][1].record(stream)
            torch.cuda.synchronize()
        clk.mark_end()
    launches = (_lib.launch_count() - launches0) // total
    dev_us = [evs[k][0].elapsed_time(evs[k][1]) * 1000.0 for k in range(warmup, total)]
    # end-to-end through the public host API (each tick: H2D inputs, kernels, D2H results)
    eng2 = TickEngine(fns, tables, cluster0, cfg, scaler_interval_ms=interval_ms,
                      cold_start_ms=5000.0, pod_counter=len(cluster0.pods), device=local)
    rng = random.Random(0)
    host_arr = [arrivals_for(k) for k in range(total)]
    e2e_us, obj_us, acts = [], [], []
    for k in range(total):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        res = eng2.tick(interval_ms * (k + 1), host_arr[k], idle=None)
        t2 = time.perf_counter()
        acts.append(len(res.actions))  # the caller's ScalingAction objects (built on access)
        t3 = time.perf_counter()
        e2e_us.append((t2 - t1) * 1e6)
        obj_us.append((t3 - t1) * 1e6)
    e2e_us, obj_us = e2e_us[warmup:], obj_us[warmup:]
    acts = acts[warmup:]
    return {"functions": nfn, "gpus_simulated": ngpu, "grid": "32x91x100, delta 1" if full_grid
            else "6x10x10, delta 10", "ticks": ticks,
            "device_us_median": float(np.median(dev_us)), "device_us_max": float(np.max(dev_us)),
            "e2e_us_median": float(np.median(e2e_us)), "e2e_us_max": float(np.max(e2e_us)),
            "e2e_objects_us_median": float(np.median(obj_us)),
            "e2e_objects_us_max": float(np.max(obj_us)),
            "actions_per_tick_mean": float(np.mean(acts)), "launches_per_tick": int(launches),
            "world_build_s": round(build_s, 3), "clocks": clk.summary(),
            "e2e_api": "TickEngine.tick -> TickResult (rapp_tick_submit/collect: H2D arrivals+idle, "
                       "D2H packed actions+rates, new pod ids named); e2e_objects adds building "
                       "the caller's ScalingAction objects with their pod ids"}


def run_config1(args, local, reps=20):
    """BASELINE config 1 (the reference's CPU-runnable case): the ResNet-50 table queried
    over b = 1..32 x sm = 10..100 x quota = 1..100 (291,200 points, latency + rps) and
    most_efficient_config for 64 log-spaced targets at quota steps 1 and 10 — device time
    per sweep / per batched search, next to the reference's compiled kernel on one core."""
    import torch
    from paper_2505_01968_b200 import PerfTable, PerfTableSet
    s = list(range(10, 101, 10))
    q = list(range(10, 101, 10))
    lat = surface(*MODELS["resnet50"], BATCHES, s, q)
    t = PerfTable("resnet50", BATCHES, s, q, lat, device=local)
    b3, s3, q3 = np.meshgrid(np.arange(1, 33.0), np.arange(10, 101.0), np.arange(1, 101.0),
                             indexing="ij")
    c = np.ascontiguousarray(np.column_stack([b3.ravel(), s3.ravel(), q3.ravel()]))
    dev = torch.device("cuda", local)
    dc = torch.from_numpy(c).to(dev)
    out = torch.empty(len(c), dtype=torch.float64, device=dev)
    rps = torch.empty_like(out)
    st = torch.cuda.current_stream(dev)
    t.predict_latency_many(dc, out, rps, stream=st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        t.predict_latency_many(dc, out, rps, stream=st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    sweep_us = e0.elapsed_time(e1) * 1000.0 / reps
    peak = t.throughput(32, 100, 100)
    targets = torch.tensor(np.geomspace(0.001, 2.0 * peak, 64), dtype=torch.float64,
                           device=dev)
    search_us = {}
    for step in (1, 10):
        ts = PerfTableSet([(t, None)] * 64, quota_step=step)
        o = torch.empty((64, 3), dtype=torch.int32, device=dev)
        ts.search_dev(targets, o)
        e0.record(st)
        for _ in range(reps):
            ts.search_dev(targets, o, stream=st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        search_us[f"quota_step_{step}"] = e0.elapsed_time(e1) * 1000.0 / reps
    ref = None
    try:
        from oracle.binding import load_reference_kernel
        k = load_reference_kernel()
        if k is not None:
            o2 = np.empty(len(c))
            t0 = time.perf_counter()
            k.interp3_many(t._b_axis, t._s_axis, t._q_axis, t.latency_ms, c, o2)
            ref = {"sweep_us": (time.perf_counter() - t0) * 1e6, "cores": 1,
                   "kind": "reference", "what": "the reference's compiled interp3_many"}
    except Exception:  # noqa: BLE001 — the baseline is optional on a box without oracle/_ref
        ref = None
    return {"points": len(c), "sweep_us_device": sweep_us,
            "sweep_predictions_per_s": len(c) / (sweep_us * 1e-6),
            "search_64_targets_us_device": search_us, "cpu_baseline": ref}


def run_replay(args, local, name="burst-100", reps=3):
    """Config 3: the 100-function burst trace replay captured from the reference simulator
    (tests/golden/replay.json): every scaler tick through the public host API —
    TickEngine.release (the simulator's between-tick releases) + TickEngine.tick (H2D
    arrivals and idle flags, kernels, D2H actions and rates) — timed end to end per tick.
    Decisions are checked against the capture on every tick."""
    import torch
    from paper_2505_01968_b200 import PerfTable
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    from paper_2505_01968_b200.tick import TickEngine
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_io import cluster_from, function_from, fx
    with open(os.path.join(ROOT, "tests", "golden", "replay.json")) as fh:
        run = next(r for r in json.load(fh)["runs"] if r["name"] == name)
    fns = [function_from(f) for f in run["functions"]]
    tables = {}
    for tn, t in run["tables"].items():
        b, s_, q = (np.asarray(t[k], dtype=np.float64) for k in ("batches", "sms", "quotas"))
        v = np.array([float.fromhex(x) for x in t["latency_ms"]]).reshape(len(b), len(s_), len(q))
        tables[tn] = PerfTable(t["function_id"], t["batches"], t["sms"], t["quotas"], v,
                               device=local)
    cfg = ScalerConfig(alpha=fx(run["alpha"]), beta=fx(run["beta"]), delta_iq=run["delta"],
                       cooldown_ms=fx(run["cooldown_ms"]), r_min=fx(run["r_min"]))
    times = []
    eng = res = None
    for rep in range(reps):
        # the previous pass's engine (kept alive by its last TickResult) is destroyed here,
        # not inside the first timed tick of this pass
        eng = res = None
        eng = TickEngine(fns, tables, cluster_from(run["initial"]), cfg,
                         kalman_params={k: fx(v) for k, v in run["kalman"].items()},
                         scaler_interval_ms=fx(run["interval_ms"]),
                         cold_start_ms=fx(run["cold_start_ms"]),
                         pod_counter=run["pod_counter0"], policy=run["policy"], device=local)
        for t in run["ticks"]:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            eng.release(t["released"])
            res = eng.tick(fx(t["now"]), t["arrivals"], idle=set(t["idle"]))
            dt = time.perf_counter() - t0
            if rep > 0:  # the first pass warms up
                times.append(dt * 1e6)
            got = [[a.function_id, a.kind.value, a.batch, a.sm_percent, a.quota_percent,
                    a.pod_id, a.gpu_id] for a in res.actions]
            if got != [list(a) for a in t["actions"]]:
                raise RuntimeError("replay decisions differ from the reference capture")
    acts = sum(len(t["actions"]) for t in run["ticks"])
    return {"functions": len(fns), "gpus_simulated": len(run["initial"]["gpus"]),
            "ticks": len(run["ticks"]), "actions": acts, "passes_timed": reps - 1,
            "e2e_us_median": float(np.median(times)), "e2e_us_max": float(np.max(times)),
            "decisions": "identical to the reference simulator on every tick",
            "api": "TickEngine.release + TickEngine.tick (host arrays, idle pod ids)"}


def reference_package():
    """The reference package `hybridscale` (baseline/_ref, installed by baseline/install.sh;
    it travels to the GPU box with the snapshot), or None."""
    try:
        import hybridscale
        return hybridscale
    except ImportError:
        return None


def reference_config4_sample(full_grid=False, sample=40):
    """The reference's own SimulationEngine._handle_scaler (hs/sim.py:470-491) on the
    config-4 world (1,000 functions, 400 GPUs, the bench's first tick of load), restricted
    to the first `sample` functions in its sorted tick order while the cluster keeps all
    1,000 functions' pods (each decision deep-copies the whole cluster, hs/autoscaler.py:111).
    Seconds per tick extrapolated linearly to 1,000 functions, labelled as such."""
    hs = reference_package()
    if hs is None:
        return None
    from hybridscale import (FunctionSpec, PerfTable, PodConfig, PodInstance, PodState,
                             ScalerConfig, SimConfig, WorkloadTrace, allocator)
    from hybridscale.sim import SimulationEngine, _PodRuntime, build_cluster
    nfn, ngpu = 1000, 400
    rng = random.Random(0)  # the same draws as make_config4_world
    if full_grid:
        bs, ss, qs = list(range(1, 33)), list(range(10, 101)), list(range(1, 101))
    else:
        bs, ss, qs = BATCHES, list(range(10, 101, 10)), list(range(10, 101, 10))
    fns, tables, caps = [], {}, {}
    for i in range(nfn):
        fid = f"fn-{i:04d}"
        fixed, per, floor = rng.uniform(4, 20), rng.uniform(0.5, 4), rng.uniform(0.2, 0.4)
        lat = surface(fixed, per, floor, 1.0 - floor, bs, ss, qs)
        tables[fid] = PerfTable(fid, bs, ss, qs, lat)
        fns.append(FunctionSpec(function_id=fid, baseline_latency_ms=20.0, perf_table_ref=fid,
                                allowed_batches=list(BATCHES), initial=PodConfig(8, 20, 20)))
        caps[fid] = 8 / (float(lat[bs.index(8), ss.index(20), qs.index(20)]) / 1000.0)
    cluster = build_cluster(ngpu, functions=fns)
    for i, f in enumerate(fns):
        allocator.place_pod(cluster, PodInstance(f"pod-{i:06d}", f.function_id, 8, 20, 20, "",
                                                 state=PodState.RUNNING), f"gpu-{i % ngpu:03d}")
    eng = SimulationEngine(WorkloadTrace(entries=[], horizon_ms=1.0), fns, tables, cluster,
                           ScalerConfig(delta_iq=1 if full_grid else 10),
                           SimConfig(scaler_interval_ms=2000.0, cold_start_ms=5000.0),
                           "hybrid", None)
    for pod in cluster.pods.values():  # what _bootstrap does for its own placements
        pod.capability_rps = eng._capability(pod)
        eng._runtimes[pod.pod_id] = _PodRuntime(pod)
        eng._open_cost_interval(pod, 0.0)
    eng._pod_counter = len(cluster.pods)
    arrivals = config4_arrivals(fns, caps, rng, 2.0, 0.0, 3.0)  # the bench's first tick
    for fid, a in arrivals.items():
        eng._tick_arrivals[fid] = a
    keep = sorted(eng.functions)[:sample]
    eng.functions = {fid: eng.functions[fid] for fid in keep}
    t0 = time.perf_counter()
    eng._handle_scaler(2000.0)
    dt = time.perf_counter() - t0
    return {"value": dt * nfn / sample * 1e6, "unit": "us/tick", "cores": 1,
            "kind": "reference",
            "sample": f"hybridscale SimulationEngine._handle_scaler over the first {sample} of "
                      f"{nfn} functions of tick 1 ({dt:.2f} s, whole 400-GPU cluster), "
                      f"extrapolated x{nfn // sample}"}


def reference_config3(local, policy="hybrid"):
    """Config 3 (100 functions, 60 s burst replay, 64 GPUs, tests/experiments.py) simulated
    twice: by the unmodified reference (`hybridscale.sim.run`) and by the drop-in
    (`integration.hybridscale_b200.run`: the same simulator with its per-tick hook
    `_handle_scaler` running one device tick).  Returns µs per `_handle_scaler` call of both
    and whether the four metric CSVs (hs/sim.py:651-685) are byte-identical."""
    hs = reference_package()
    if hs is None:
        return None
    import tempfile
    from hybridscale.sim import SimulationEngine
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import experiments as ex
    from integration.hybridscale_b200 import B200SimulationEngine
    from integration.hybridscale_b200 import run as b200_run
    spec = ex.config3_runs(hs, policies=(policy,))[0]
    times = {"reference": [], "b200": []}
    orig_ref, orig_b200 = SimulationEngine._handle_scaler, B200SimulationEngine._handle_scaler

    def timed(orig, bucket):
        def handle(self, now):
            t0 = time.perf_counter()
            orig(self, now)
            times[bucket].append((time.perf_counter() - t0) * 1e6)
        return handle
    digests = {}
    try:
        B200SimulationEngine._handle_scaler = timed(orig_b200, "b200")
        with tempfile.TemporaryDirectory() as d:
            digests["b200"] = ex.digest(ex.run_to_csvs(
                lambda *a: b200_run(*a, device=local), spec, d))
        SimulationEngine._handle_scaler = timed(orig_ref, "reference")
        B200SimulationEngine._handle_scaler = orig_b200  # only the base class is timed now
        with tempfile.TemporaryDirectory() as d:
            from hybridscale.sim import run as ref_run
            digests["reference"] = ex.digest(ex.run_to_csvs(ref_run, spec, d))
    finally:
        SimulationEngine._handle_scaler = orig_ref
        B200SimulationEngine._handle_scaler = orig_b200
    # the first B200 tick uploads the world (TickEngine construction)
    b = times["b200"][1:]
    r = times["reference"]
    return {"ticks": len(r), "b200_us_median": float(np.median(b)),
            "b200_us_max": float(np.max(b)), "ref_us_median": float(np.median(r)),
            "ref_us_max": float(np.max(r)),
            "csv_identical": digests["b200"] == digests["reference"]}


def tick_cpu_baseline(args, nticks=2):
    """The scaler oracle (pure-Python restatement of the reference tick, oracle/) on one
    host core for the same config-4 world: seconds per tick.  The reference itself spends
    ~44 s/tick here (>98% in copy.deepcopy); the restatement copies less."""
    import copy
    from oracle import scaler_oracle as so
    from paper_2505_01968_b200.core import PodInstance, PodState, SmPartition
    fns, tables, cluster, caps = make_config4_world(1000, 400, seed=0)
    otables = {k: so.OTable(t) for k, t in tables.items()}
    cfg = {"alpha": 0.9, "beta": 0.5, "delta": 10, "cooldown_ms": 30000.0, "r_min": 1.0}
    kal = {"A": 1.0, "Q": 4.0, "H": 1.0, "D": 16.0}
    functions = {f.function_id: f for f in fns}
    rng = random.Random(0)
    kstate, last_down, counter = {}, {}, len(cluster.pods)
    times = []
    for k in range(nticks):
        swing = (1.0, 1.5, 0.2, 2.0, 0.05)[k % 5]
        arr = config4_arrivals(fns, caps, rng, 2.0, 0.0, 3.0 * swing)
        t0 = time.perf_counter()
        _, _, _, counter = so.tick(
            cfg, functions, otables, cluster, 2000.0 * (k + 1), 2000.0, arr, set(cluster.pods),
            kstate, kal, 1.0, last_down, counter,
            lambda pid, fid, b, s, q, g: PodInstance(pid, fid, b, s, q, g,
                                                     state=PodState.COLD_STARTING),
            lambda sm: SmPartition(sm), cold_start_ms=5000.0)
        times.append(time.perf_counter() - t0)
    return {"value": float(np.median(times)) * 1e6, "unit": "us/tick", "cores": 1,
            "kind": "port", "sample": f"{nticks} config-4 ticks of oracle/scaler_oracle.py "
            "(1,000 functions, 400 GPUs)"}


# ----------------------------------------------------------------------------------------
# CPU baseline / reference arm: the reference's own compiled kernel on all host cores
# ----------------------------------------------------------------------------------------

_W = {}


def _worker_init(rows, seed):
    from oracle.binding import load_oracle, load_reference_kernel
    ref = load_reference_kernel()
    if ref is not None:
        fn, kind = ref.interp3_many, "reference"
    else:
        from oracle.binding import or_interp3_many

        def fn(b, s, q, v, c, out):
            out[:] = or_interp3_many(b, s, q, v, c)
        load_oracle()
        kind = "port"
    arrays = config2_arrays()
    rng = np.random.default_rng(seed + os.getpid())
    work = []
    for _, b, s, q, v in arrays:
        c = np.column_stack([rng.uniform(b[0], b[-1], rows), rng.uniform(s[0], s[-1], rows),
                             rng.uniform(q[0], q[-1], rows)])
        work.append((b, s, q, v, np.ascontiguousarray(c), np.empty(rows)))
    _W.update(fn=fn, kind=kind, work=work)


def _worker_run(_):
    for b, s, q, v, c, out in _W["work"]:
        _W["fn"](b, s, q, v, c, out)
    return _W["kind"]


def host_cores():
    try:
        return len(_ALL_CPUS or os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_reference(steps, warmup, rows_per_model=1_000_000, procs=None):
    """Times the reference kernel over a process pool; returns (predictions/s, info)."""
    import multiprocessing as mp
    procs = procs or host_cores()
    ctx = mp.get_context("spawn")  # the parent holds a CUDA context: never fork it
    with ctx.Pool(procs, initializer=_worker_init, initargs=(rows_per_model, 12345)) as pool:
        kinds = pool.map(_worker_run, range(procs))
        for _ in range(max(0, warmup - 1)):
            pool.map(_worker_run, range(procs))
        t0 = time.perf_counter()
        for _ in range(steps):
            pool.map(_worker_run, range(procs))
        dt = time.perf_counter() - t0
    preds = steps * procs * len(MODELS) * rows_per_model
    kind = kinds[0]
    sample = (f"{len(MODELS)} config-2 tables x {rows_per_model} queries/process/step, "
              f"{procs} procs, {steps} steps ({dt:.2f} s)")
    return preds / dt, {"kind": kind, "cores": procs, "sample": sample}


# ----------------------------------------------------------------------------------------


def split_check(rank, world, local):
    """shard.search_split — one config-2 lattice (32 x 100 x 100 at quota step 1) split
    over the ranks by batch slabs, meet keys combined by an NCCL all-reduce MIN (fallback:
    all-gather) — equals the unsplit device search on every rank, for feasible, boundary and
    unreachable targets."""
    from paper_2505_01968_b200 import PerfTable
    from paper_2505_01968_b200.shard import search_split
    name, b, s, q, v = config2_arrays()[0]
    t = PerfTable(name, BATCHES, list(range(1, 101)), list(range(1, 101)), v, device=local)
    top = max_lattice_rps(t)
    ok = True
    for target in (0.5, 0.1 * top, 0.5 * top, top, 2.0 * top):
        for step, allowed in ((1, list(range(1, 33))), (10, None)):
            got = search_split(t, target, rank, world, quota_step=step, batches=allowed)
            ok &= got == t.most_efficient_config(target, quota_step=step, batches=allowed)
    return bool(ok)


def self_launch(argv, gpus):
    """`bench.py --gpus N` outside torchrun: relaunch as N ranks (one process per GPU) with
    torch.distributed.run on 127.0.0.1 and pass its exit code through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *argv]
    return subprocess.run(cmd).returncode


def _r(x, nd=1):
    return None if x is None else round(float(x), nd)


def tick_summary(t, ref=None):
    """Compact driver-visible summary of one tick workload (µs per tick)."""
    out = {"dev_med": _r(t["device_us_median"]), "dev_max": _r(t["device_us_max"]),
           "e2e_med": _r(t["e2e_us_median"]), "e2e_max": _r(t["e2e_us_max"]),
           "acts": _r(t["actions_per_tick_mean"]), "ticks": t["ticks"]}
    if "e2e_objects_us_median" in t:
        out["obj_med"] = _r(t["e2e_objects_us_median"])
        out["obj_max"] = _r(t["e2e_objects_us_max"])
    if ref is not None:
        out["ref_us"] = _r(ref["value"], 0)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["stream", "lattice", "tick", "mlp"], default="stream")
    ap.add_argument("--ticks", type=int, default=50)
    ap.add_argument("--full-grid", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--queries", type=int, default=QUERIES_PER_MODEL)
    ap.add_argument("--functions", type=int, default=3125)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--detail", default=None,
                    help="also write the full (uncompacted) result JSON to this path")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(sys.argv[1:], args.gpus))

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        if rank != 0:
            return
        # each step is a bounded sample (~0.5 s of work per host core) of the workload
        value, info = cpu_reference(args.steps, args.warmup, rows_per_model=250_000)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "impl": "reference",
                "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "config2 4-model sweep (bounded CPU sample per step)",
                           "parallelism": f"{info['cores']} host processes"},
                "cpu_baseline": {"value": value, "unit": UNIT, **info},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    rank, world, local = dist_init(args.gpus)
    detail = {}
    if args.workload == "tick":
        tick = run_tick(args, local, full_grid=args.full_grid)
        line = None
        if rank == 0:
            line = {"metric": METRIC, "value": tick["device_us_median"], "unit": "us/tick",
                    "n_gpus": world, "steps": tick["ticks"], "warmup": 3,
                    "ms_per_step": tick["device_us_median"] / 1000.0, "higher_is_better": False,
                    "scaling": "replicas", "vs_baseline": None, "dtype": "f64",
                    "data": "synthetic", "config": {"workload": "config4 tick: " + tick["grid"]},
                    "e2e": {"value": tick["e2e_us_median"], "unit": "us/tick",
                            "h2d_bytes_per_step": 1000 * 8 + 1000,
                            "d2h_bytes_per_step": "actions (32 B each) + 2 x 8 KB rates"},
                    "tick": tick_summary(tick),
                    "cpu_baseline": reference_config4_sample(args.full_grid)
                    or tick_cpu_baseline(args),
                    "gpu_launches": tick["launches_per_tick"] * tick["ticks"],
                    "clocks": tick["clocks"], "impl": "ours"}
            detail = {"tick": tick}
        finish(line, detail, args, world)
        return
    if args.workload == "mlp":
        res = run_mlp(args, rank, world, local)
        line = None
        if rank == 0:
            line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world,
                    "steps": res["steps"], "warmup": args.warmup,
                    "ms_per_step": res["ms"] / res["steps"], "higher_is_better": True,
                    "scaling": res["scaling"], "vs_baseline": None, "dtype": res["dtype"],
                    "data": "synthetic", "config": res["config"], "roofline": res["roofline"],
                    "cpu_baseline": res["cpu_baseline"], "e2e": res["e2e"],
                    "gpu_launches": res["launches"], "clocks": res["clocks"], "impl": "ours",
                    "search": res["search"]}
        finish(line, detail, args, world)
        return
    res = (run_stream if args.workload == "stream" else run_lattice)(args, rank, world, local)
    sharded = None
    if world > 1 and args.workload == "stream" and not args.no_extra:
        # the N>1 line also runs the config-5 search sharded over the ranks: per-rank
        # function blocks + one NCCL all-gather of the decisions (and a giant-lattice split
        # check: batch slabs, all-reduce MIN of packed keys)
        largs = argparse.Namespace(**{**vars(args), "steps": 20, "functions": 3125,
                                      "no_e2e": True})
        lat = run_lattice(largs, rank, world, local)
        sharded = {"value": lat["value"], "ms_per_step": _r(lat["ms"] / largs.steps, 4),
                   "frac": lat["roofline"]["frac"], "split_ok": split_check(rank, world, local),
                   "workload": "config5 3125 fn, functions sharded, NCCL all_gather",
                   "scaling": "strong"}
    if rank != 0:
        finish(None, None, args, world)
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline and args.workload == "stream":
        with all_cpus():
            v, info = cpu_reference(steps=3, warmup=1)
        cpu = {"value": v, "unit": UNIT, **info}
    if world == 1 and not args.no_cpu_baseline and args.workload == "lattice":
        with all_cpus():
            cpu = lattice_cpu_baseline()
    line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms"] / args.steps,
            "higher_is_better": True, "scaling": res["scaling"], "vs_baseline": None,
            "dtype": res["dtype"], "data": "synthetic", "config": res["config"],
            "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": res["e2e"],
            "gpu_launches": res["launches"], "clocks": res["clocks"], "impl": "ours"}
    if sharded is not None:
        line["sharded_search"] = sharded
        line["comm"] = {"backend": "nccl", "nranks": world}
    if world == 1 and args.workload == "stream" and not args.no_extra:
        # the second half of the metric ("scaling decisions/tick latency") and config 5;
        # compact summaries on the line, everything else in the detail record
        t4 = run_tick(args, local, ticks=20)
        t4f = run_tick(args, local, ticks=20, full_grid=True)
        t3 = run_tick(args, local, ticks=20, nfn=100, ngpu=64)
        rep = run_replay(args, local)
        c3 = reference_config3(local)
        r4 = reference_config4_sample(False)
        r4f = reference_config4_sample(True)
        c1 = run_config1(args, local)
        largs = argparse.Namespace(**{**vars(args), "steps": 50, "functions": 3125})
        lat = run_lattice(largs, rank, world, local)
        lcpu = lattice_cpu_baseline_all()
        margs = argparse.Namespace(**{**vars(args), "steps": 30, "queries": 25_000_000})
        mlp = run_mlp(margs, rank, world, local)
        ticks = {"config4": tick_summary(t4, r4), "config4_full_grid": tick_summary(t4f, r4f),
                 "config3_size": tick_summary(t3),
                 "replay_config3": {"tick_e2e_med": _r(rep["e2e_us_median"]),
                                    "tick_e2e_max": _r(rep["e2e_us_max"])}}
        if c3 is not None:
            ticks["replay_config3"].update(
                {"dropin_med": _r(c3["b200_us_median"]), "dropin_max": _r(c3["b200_us_max"]),
                 "ref_med": _r(c3["ref_us_median"], 0), "ref_max": _r(c3["ref_us_max"], 0),
                 "csv_identical": c3["csv_identical"]})
        line["ticks"] = ticks
        line["ticks_unit"] = "us/tick; dev=CUDA events, e2e=TickEngine.tick, obj=e2e + the " \
                             "ScalingAction objects, dropin=" \
                             "B200SimulationEngine._handle_scaler, ref=hybridscale " \
                             "_handle_scaler (config4: 40-fn sample x25)"
        line["lattice_config5"] = {"value": lat["value"], "ms_per_step": _r(lat["ms"] / 50, 4),
                                   "frac": lat["roofline"]["frac"],
                                   "e2e": _r(lat["e2e"]["value"], -6) if lat["e2e"] else None,
                                   "cpu": _r(lcpu["value"], -3)}
        line["learned_mlp"] = {"value": mlp["value"], "frac": mlp["roofline"]["frac"]}
        line["config1_sweep_us"] = _r(c1["sweep_us_device"], 2)
        detail = {"tick_config4": t4, "tick_config4_full_grid": t4f, "tick_config3_size": t3,
                  "replay_config3": rep, "reference_config3": c3,
                  "reference_config4": [r4, r4f], "config1": c1, "lattice_config5": lat,
                  "lattice_cpu": lcpu, "learned_mlp": mlp,
                  "tick_port_baseline": tick_cpu_baseline(args)}
    finish(line, detail, args, world)


def finish(line, detail, args, world):
    """Rank 0 prints ONE compact JSON line last (after the process group is torn down, so
    no later log line follows it); the full record goes to --detail and to stderr."""
    if world > 1:
        import torch.distributed as dist
        barrier(world)
        dist.destroy_process_group()
    if line is None:
        return
    if detail:
        full = {"line": line, "detail": detail}
        if args.detail:
            with open(args.detail, "w") as fh:
                json.dump(full, fh, default=str)
        print("bench detail: " + json.dumps(detail, default=str), file=sys.stderr, flush=True)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
