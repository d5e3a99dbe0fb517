"""Host-path overhead of a config-4 tick: two identical engines run the same ticks, one
through TickEngine.tick (host arrays in, actions out) and one through rapp_tick_run_dev on
resident inputs followed by a stream synchronise; both timed by the host clock.

    python tools/tick_host_overhead.py [--full-grid]
"""
import copy
import ctypes
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_01968_b200 import _lib  # noqa: E402
from paper_2505_01968_b200.autoscaler import ScalerConfig  # noqa: E402
from paper_2505_01968_b200.tick import TickEngine  # noqa: E402

full = "--full-grid" in sys.argv
fns, tables, cluster, caps = bench.make_config4_world(1000, 400, seed=0, full_grid=full,
                                                      device=0)
cluster2 = copy.deepcopy(cluster)
cfg = ScalerConfig(delta_iq=1 if full else 10)
kw = dict(scaler_interval_ms=2000.0, cold_start_ms=5000.0, pod_counter=len(cluster.pods),
          device=0)
eng = TickEngine(fns, tables, cluster, cfg, **kw)
eng2 = TickEngine(fns, tables, cluster2, cfg, **kw)
eng3 = TickEngine(fns, tables, copy.deepcopy(cluster2), cfg, **kw)
eng._all_idle = np.ones(1 << 20, dtype=np.uint8)  # every pod idle, as d_idle below
lib = _lib.load()
rng = random.Random(0)
order = sorted(fns, key=lambda f: f.function_id)
d_idle = torch.ones(1 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
host, dev, call, full = [], [], [], []
for k in range(25):
    swing = (1.0, 1.5, 0.2, 2.0, 0.05)[k % 5]
    a = bench.config4_arrivals(fns, caps, rng, 2.0, 0.0, 3.0 * swing)
    arr = np.array([a[f.function_id] for f in order], dtype=np.int64)
    d_arr = torch.from_numpy(arr).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(lib.rapp_tick_run_dev(eng2._h, 2000.0 * (k + 1), d_arr.data_ptr(),
                                     d_idle.data_ptr(), st.cuda_stream))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    nact = ctypes.c_int64()
    t2 = time.perf_counter()
    rc = lib.rapp_tick_run(eng._h, 2000.0 * (k + 1), _lib.i64ptr(arr), eng._all_idle.ctypes.data,
                           None,
                           eng._act_buf.ctypes.data, len(eng._act_buf), ctypes.byref(nact),
                           eng._obs.ctypes.data, eng._pred.ctypes.data)
    t3 = time.perf_counter()
    _lib.check(rc)
    eng.counter += int((eng._act_buf[:nact.value]["kind"] == 2).sum())
    t4 = time.perf_counter()
    eng3.tick(2000.0 * (k + 1), arr, idle=None)
    t5 = time.perf_counter()
    if k >= 5:
        dev.append((t1 - t0) * 1e6)
        call.append((t3 - t2) * 1e6)
        full.append((t5 - t4) * 1e6)
print(f"run_dev+sync median {np.median(dev):7.1f} us   rapp_tick_run (C ABI) median "
      f"{np.median(call):7.1f} us   difference {np.median(np.array(call) - np.array(dev)):6.1f} us")
for name, xs in (("run_dev+sync", dev), ("C ABI call", call), ("TickEngine.tick", full)):
    print(f"{name:16s} median {np.median(xs):7.1f}  max {np.max(xs):7.1f} us")
i = int(np.argmax(dev))
print(f"heaviest tick: run_dev+sync {dev[i]:.1f}, C ABI {call[i]:.1f}, TickEngine.tick {full[i]:.1f} us")
