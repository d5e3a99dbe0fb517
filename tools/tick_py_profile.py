"""Where TickEngine.tick's host-side Python time goes (config-4 full-grid ticks): wall time
of the C-ABI call vs the wrapper around it, per tick, with the wrapper's parts timed.

    python tools/tick_py_profile.py [--full-grid]"""
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
eng = TickEngine(fns, tables, cluster, ScalerConfig(delta_iq=1 if full else 10),
                 scaler_interval_ms=2000.0, cold_start_ms=5000.0,
                 pod_counter=len(cluster.pods), device=0)
lib = _lib.load()
real_run = lib.rapp_tick_run
t_call = []


def timed_run(*a):
    t0 = time.perf_counter()
    rc = real_run(*a)
    t_call.append(time.perf_counter() - t0)
    return rc


lib.rapp_tick_run = timed_run
real_book = eng._bookkeep
t_book = []


def timed_book(raw):
    t0 = time.perf_counter()
    r = real_book(raw)
    t_book.append(time.perf_counter() - t0)
    return r


eng._bookkeep = timed_book
rng = random.Random(0)
order = sorted(fns, key=lambda f: f.function_id)
rows = []
for k in range(30):
    swing = (1.0, 1.5, 0.2, 2.0, 0.05)[k % 5]
    a = bench.config4_arrivals(fns, caps, rng, 2.0, 0.0, 3.0 * swing)
    arr = np.array([a[f.function_id] for f in order], dtype=np.int64)
    t0 = time.perf_counter()
    res = eng.tick(2000.0 * (k + 1), arr, idle=None)
    tot = time.perf_counter() - t0
    if k >= 3:
        rows.append((tot * 1e6, t_call[-1] * 1e6, t_book[-1] * 1e6, len(res.raw)))
rows.sort()
for tot, call, book, n in rows[-5:] + rows[len(rows) // 2: len(rows) // 2 + 1]:
    print(f"tick total {tot:7.1f} us  C call {call:7.1f}  bookkeep {book:6.1f}  "
          f"rest {tot - call - book:6.1f}  actions {n}")
