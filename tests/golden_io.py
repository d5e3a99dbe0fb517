"""Rebuilds golden-vector records (tests/golden/*.json) as host objects."""

from __future__ import annotations

import numpy as np

from paper_2505_01968_b200.core import (ClusterState, FunctionSpec, GpuDevice, PodConfig,
                                        PodInstance, PodState, SmPartition)


def fx(h):
    return None if h is None else float.fromhex(h)


def cluster_from(d) -> ClusterState:
    c = ClusterState(clock_ms=fx(d["clock_ms"]))
    for g in d["gpus"]:
        c.gpus[g["id"]] = GpuDevice(g["id"], partitions=[
            SmPartition(p["sm"], list(p["residents"]), p["alloc"]) for p in g["partitions"]])
    for p in d["pods"]:
        c.pods[p["id"]] = PodInstance(p["id"], p["fid"], p["b"], p["s"], p["q"], p["gpu"],
                                      state=PodState(p["state"]))
    return c


def cluster_to(c) -> dict:
    return {"gpus": [{"id": g.gpu_id, "partitions": [
                {"sm": p.sm_percent, "residents": list(p.resident_pods),
                 "alloc": p.quota_allocated} for p in g.partitions]}
                     for g in c.gpus.values()],
            "pods": sorted([p.pod_id, p.function_id, p.batch, p.sm_percent, p.quota_percent,
                            p.gpu_id, getattr(p.state, "value", p.state)]
                           for p in c.pods.values())}


def golden_cluster_to(d) -> dict:
    return {"gpus": [{"id": g["id"], "partitions": g["partitions"]} for g in d["gpus"]],
            "pods": sorted([p["id"], p["fid"], p["b"], p["s"], p["q"], p["gpu"], p["state"]]
                           for p in d["pods"])}


def function_from(d) -> FunctionSpec:
    return FunctionSpec(function_id=d["id"], baseline_latency_ms=20.0, perf_table_ref=d["table"],
                        min_rps=fx(d["min_rps"]), allowed_batches=list(d["allowed"]),
                        initial=PodConfig(*d["initial"]))


def make_pod(pid, fid, b, s, q, gpu):
    return PodInstance(pid, fid, b, s, q, gpu, state=PodState.COLD_STARTING)


def make_part(sm):
    return SmPartition(sm)


def surface_tables(tdesc, fns):
    """Tables of a tick run, rebuilt from the gen_tables-style parameters."""
    import bench
    from paper_2505_01968_b200 import PerfTable
    out = {}
    for f, (fixed, per, floor) in zip(fns, tdesc["params"]):
        fixed, per, floor = fx(fixed), fx(per), fx(floor)
        lat = bench.surface(fixed, per, floor, 1.0 - floor, tdesc["batches"], tdesc["sms"],
                            tdesc["quotas"])
        out[f.perf_table_ref or f.function_id] = PerfTable(
            f.function_id, tdesc["batches"], tdesc["sms"], tdesc["quotas"], lat)
    return out
