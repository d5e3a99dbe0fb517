"""Cycle breakdown of the commit kernel per tick (needs a RAPP_TICK_PROF build):
    RAPP_LIB=build_variants/prof.so python tools/tick_commit_breakdown.py [--full-grid]"""
import collections
import copy
import ctypes
import os
import random
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_01968_b200 import _lib  # noqa: E402
from paper_2505_01968_b200.autoscaler import ScalerConfig  # noqa: E402
from paper_2505_01968_b200.tick import TickEngine  # noqa: E402

NAMES = ["batch wait", "vertical spec/walk", "used-GPU rest", "fresh-GPU branch",
         "scale-down", "vertical headroom", "functions (wall)", "vertical change+emit",
         "hu argmin", "hu best_slot", "hu T+covering", "hu new_pod", "hu place", "hu emit",
         "fast lanes", "fast candidates", "fast_run", "fast_run calls", "-", "runs committed",
         "prologue", "epilogue", "hu T row read", "hu new-partition slots", "hu steps", "generic ups",
         "generic ups to horizontal", "tail horizontals", "hu rows outside the mask"]
COUNTS = (14, 15, 17, 19, 23, 24, 25, 26, 27, 28)


def main(full_grid, nticks=6):
    fns, tables, cluster, caps = bench.make_config4_world(1000, 400, seed=0, device=0,
                                                          full_grid=full_grid)
    cluster2 = copy.deepcopy(cluster)
    cfg = ScalerConfig(delta_iq=1 if full_grid else 10)
    kw = dict(scaler_interval_ms=2000.0, cold_start_ms=5000.0, pod_counter=len(cluster.pods),
              device=0)
    eng = TickEngine(fns, tables, cluster, cfg, **kw)
    eng2 = TickEngine(fns, tables, cluster2, cfg, **kw)
    lib = _lib.load()
    rd = lib.rapp_tick_prof_read
    rd.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = np.zeros(32, dtype=np.uint64)
    rd(buf.ctypes.data, 1)
    rng = random.Random(0)
    order = sorted(fns, key=lambda f: f.function_id)
    for k in range(nticks):
        swing = (1.0, 1.5, 0.2, 2.0, 0.05)[k % 5]
        a = bench.config4_arrivals(fns, caps, rng, 2.0, 0.0, 3.0 * swing)
        host = np.array([a[f.function_id] for f in order], dtype=np.int64)
        rd(buf.ctypes.data, 1)  # reset
        res = eng.tick(2000.0 * (k + 1), host)
        rd(buf.ctypes.data, 1)
        eng2.tick(2000.0 * (k + 1), host)
        mix = collections.Counter(str(x.kind).split(".")[-1] for x in res.actions)
        us = buf.astype(np.float64) / 1.9e3
        for i in COUNTS:
            us[i] = buf[i]  # counts, not cycles
        print(f"tick {k} actions {len(res.actions)} {dict(mix)}")
        print("   " + ", ".join(f"{NAMES[i]} {us[i]:.0f}us" for i in range(len(NAMES)) if NAMES[i] != "-"))


if __name__ == "__main__":
    main("--full-grid" in sys.argv)
