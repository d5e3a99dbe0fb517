"""Splits TickEngine.tick's end-to-end time (config 4) into the C-ABI halves (submit: H2D +
launches; collect: wait + D2H), the name-cache top-up between them, the host bookkeeping of
new pod ids and the reference-shaped action list; prints the heaviest ticks' rows too.

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
parts = {"pre": [], "submit": [], "topup": [], "collect": [], "bookkeep": [], "actions": [],
         "total": [], "nact": []}
orig_book = eng._bookkeep
orig_top = eng._top_up_names
lib = _lib.load()
orig_sub, orig_col = lib.rapp_tick_submit, lib.rapp_tick_collect
T = {}


def timed(name, fn):
    def w(*a):
        T[name + "0"] = time.perf_counter()
        r = fn(*a)
        T[name + "1"] = time.perf_counter()
        return r
    return w


lib.rapp_tick_submit = timed("s", orig_sub)
lib.rapp_tick_collect = timed("c", orig_col)
eng._top_up_names = timed("u", orig_top)
for k in range(int(os.environ.get('TICKS', '45'))):
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
        parts["pre"].append((T["s0"] - t0) * 1e6)
        parts["submit"].append((T["s1"] - T["s0"]) * 1e6)
        parts["topup"].append((T["u1"] - T["u0"]) * 1e6)
        parts["collect"].append((T["c1"] - T["c0"]) * 1e6)
        parts["nact"].append(n)
        parts["bookkeep"].append((t["b1"] - t["b0"]) * 1e6)
        parts["actions"].append((t2 - t1) * 1e6)
        parts["total"].append((t2 - t0) * 1e6)
for kname, v in parts.items():
    print(f"{kname:9s} median {np.median(v):8.1f} us  max {np.max(v):8.1f} us")
order_t = np.argsort(parts["total"])[::-1][:6]
print("heaviest ticks: " + " ".join(f"{k:>9s}" for k in parts))
for i in order_t:
    print("               " + " ".join(f"{parts[k][i]:9.1f}" for k in parts))
