"""Per-call cost of the scalar seams (SURVEY §8(b) seams 2 and 3) against the reference:
PerfTable.predict_latency / throughput / most_efficient_config and policy.decide, µs per
call, on the demo tables and a config-3 cluster (64 GPUs, 100 functions).

    python tools/seam_costs.py        (needs baseline/_ref and a GPU)"""
import copy
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))
import hybridscale as hs  # noqa: E402
import experiments as ex  # noqa: E402

from paper_2505_01968_b200 import PerfTable  # noqa: E402
from paper_2505_01968_b200.autoscaler import HybridPolicy  # noqa: E402


def per_call(fn, args_list, reps=3):
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        for a in args_list:
            fn(*a)
        best = min(best, (time.perf_counter() - t0) / len(args_list))
    return best * 1e6


def main():
    out = {}
    spec = ex.config3_runs(hs, policies=("hybrid",))[0]
    _, _, _, fns, tables, cluster_f, scaler, _, _ = spec
    t_ref = tables[fns[0].function_id]
    t_b2 = PerfTable(t_ref.function_id, t_ref.batches, t_ref.sms, t_ref.quotas, t_ref.latency_ms)
    rng = np.random.default_rng(0)
    pts = [(int(rng.choice(t_ref.batches)), int(rng.integers(10, 101)), int(rng.integers(1, 101)))
           for _ in range(2000)]
    for name in ("predict_latency", "throughput"):
        r = per_call(getattr(t_ref, name), pts)
        b = per_call(getattr(t_b2, name), pts)
        assert [getattr(t_ref, name)(*p) for p in pts[:200]] == \
            [getattr(t_b2, name)(*p) for p in pts[:200]]
        out[name] = {"reference_us": round(r, 2), "b200_us": round(b, 2)}
    targets = [(float(x),) for x in np.geomspace(1.0, 2000.0, 200)]
    r = per_call(lambda tg: t_ref.most_efficient_config(tg, quota_step=10), targets)
    b = per_call(lambda tg: t_b2.most_efficient_config(tg, quota_step=10), targets)
    out["most_efficient_config"] = {"reference_us": round(r, 2), "b200_us": round(b, 2)}
    # policy.decide on a config-3 cluster (64 GPUs, 100 functions, one pod each)
    cl = cluster_f()
    from hybridscale import allocator
    from hybridscale.core import PodInstance, PodState
    for i, f in enumerate(fns):
        allocator.place_pod(cl, PodInstance(f"pod-{i:06d}", f.function_id, f.initial.batch,
                                            f.initial.sm_percent, f.initial.quota_percent, "",
                                            state=PodState.RUNNING), f"gpu-{i % 64:03d}")
    ref_pol = hs.policies.HybridPolicy(scaler, tables)
    b2_pol = HybridPolicy(scaler, tables)
    calls = []
    for i, f in enumerate(fns[:40]):
        cap = t_ref.throughput(f.initial.batch, f.initial.sm_percent, f.initial.quota_percent)
        calls.append((f, cl, float((0.1, 1.0, 3.0, 0.05)[i % 4] * cap)))
    for f, c, rate in calls[:8]:
        assert ref_pol.decide(f, copy.deepcopy(c), rate) == b2_pol.decide(f, c, rate)
    out["HybridPolicy.decide (64 GPUs)"] = {"reference_us": round(per_call(ref_pol.decide, calls, 2), 1),
                                            "b200_us": round(per_call(b2_pol.decide, calls, 2), 1)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
