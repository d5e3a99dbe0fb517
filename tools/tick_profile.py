"""Per-tick device time of the config-4 tick (diagnostics): one line per tick with the
device µs (CUDA events around rapp_tick_run_dev) and the action mix of the same tick
(computed by a second engine through the host API on identical inputs)."""
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


def main(nticks=30, nfn=1000, ngpu=400, full_grid=False):
    fns, tables, cluster, caps = bench.make_config4_world(nfn, ngpu, seed=0, device=0,
                                                          full_grid=full_grid)
    cluster2 = copy.deepcopy(cluster)
    cfg = ScalerConfig(delta_iq=1 if full_grid else 10)
    kw = dict(scaler_interval_ms=2000.0, cold_start_ms=5000.0, pod_counter=len(cluster.pods),
              device=0)
    eng = TickEngine(fns, tables, cluster, cfg, **kw)
    eng2 = TickEngine(fns, tables, cluster2, cfg, **kw)
    rng = random.Random(0)
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    idle = torch.ones(1 << 20, dtype=torch.uint8, device="cuda")
    order = sorted(fns, key=lambda f: f.function_id)
    for k in range(nticks):
        swing = (1.0, 1.5, 0.2, 2.0, 0.05)[k % 5]
        a = bench.config4_arrivals(fns, caps, rng, 2.0, 0.0, 3.0 * swing)
        host = np.array([a[f.function_id] for f in order], dtype=np.int64)
        arr = torch.from_numpy(host).cuda()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        _lib.check(lib.rapp_tick_run_dev(eng._h, 2000.0 * (k + 1), arr.data_ptr(),
                                         idle.data_ptr(), stream.cuda_stream))
        e1.record(stream)
        torch.cuda.synchronize()
        res = eng2.tick(2000.0 * (k + 1), host, idle=None)
        mix = collections.Counter(str(x.kind).split(".")[-1] for x in res.actions)
        print(f"tick {k:3d} swing {swing:4.2f} device {e0.elapsed_time(e1) * 1000:8.1f} us "
              f"actions {len(res.actions):4d} {dict(mix)}", flush=True)


if __name__ == "__main__":
    main(nticks=int(os.environ.get("TICKS", "30")), full_grid="--full-grid" in sys.argv)
