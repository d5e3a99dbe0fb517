import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2505_01968_b200 import PerfTable, kernels
from oracle.binding import or_interp3_many
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dev = torch.device("cuda", 0)
for mi, (name, b, s, q, v) in enumerate(bench.config2_arrays()):
    t = PerfTable(name, bench.BATCHES, list(range(1, 101)), list(range(1, 101)), v)
    c = bench.gen_queries(b, s, q, n, mi, dev)
    d_out = t.predict_latency_many(c).cpu().numpy()
    hc = c.cpu().numpy()
    h_out = np.empty(n)
    kernels.interp3_many(b, s, q, v, hc, h_out)
    ref = or_interp3_many(b, s, q, v, hc)
    bd = np.nonzero(d_out.view(np.int64) != ref.view(np.int64))[0]
    bh = np.nonzero(h_out.view(np.int64) != ref.view(np.int64))[0]
    print(name, "device mismatches", len(bd), "host mismatches", len(bh))
    for idx in list(bd[:3]) + list(bh[:3]):
        print("  row", idx, hc[idx].tolist(), "dev", d_out[idx], "host", h_out[idx], "ref", ref[idx])
