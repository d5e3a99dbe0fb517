"""Splits TickEngine.tick's end-to-end time (config 4) into the C-ABI call (H2D, kernels,
D2H), the host bookkeeping of new pod ids and the reference-shaped action list.

    python tools/tick_e2e_split.py [--full-grid]
"""
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2505_01968_b200 import _lib, tick as tickmod  # noqa: E402
from paper_2505_01968_b200.autoscaler import ScalerConfig  # noqa: E402
from paper_2505_01968_b200.tick import TickEngine  # noqa: E402

full = "--full-grid" in sys.argv
fns, tables, cluster, caps = bench.make_config4_world(1000, 400, seed=0, full_grid=full,
                                                      device=0)
cfg = ScalerConfig(delta_iq=1 if full else 10)
eng = TickEngine(fns, tables, cluster, cfg, scaler_interval_ms=2000.0, cold_start_ms=5000.0,
                 pod_counter=len(cluster.pods), device=0)
rng = random.Random(0)
order = sorted(fns, key=lambda f: f.function_id)
parts = {"call": [], "bookkeep": [], "actions": [], "total": []}
orig_book = eng._bookkeep
for k in range(25):
    swing = (1.0, 1.5, 0.2, 2.0, 0.05)[k % 5]
    a = bench.config4_arrivals(fns, caps, rng, 2.0, 0.0, 3.0 * swing)
    arr = np.array([a[f.function_id] for f in order], dtype=np.int64)
    t = {}

    def book(raw):
        t["b0"] = time.perf_counter()
        r = orig_book(raw)
        t["b1"] = time.perf_counter()
        return r
    eng._bookkeep = book
    t0 = time.perf_counter()
    res = eng.tick(2000.0 * (k + 1), arr, idle=None)
    t1 = time.perf_counter()
    n = len(res.actions)
    t2 = time.perf_counter()
    if k >= 5:
        parts["call"].append((t["b0"] - t0) * 1e6)
        parts["bookkeep"].append((t["b1"] - t["b0"]) * 1e6)
        parts["actions"].append((t2 - t1) * 1e6)
        parts["total"].append((t2 - t0) * 1e6)
for kname, v in parts.items():
    print(f"{kname:9s} median {np.median(v):8.1f} us  max {np.max(v):8.1f} us")
