"""One config-2 table, N random queries through the device API (for ncu captures of K2).

    python tools/k2_probe.py [N] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_01968_b200 import PerfTable  # noqa: E402


def main(n=20_000_000, reps=3):
    name, b, s, q, v = bench.config2_arrays()[0]
    t = PerfTable(name, bench.BATCHES, list(range(1, 101)), list(range(1, 101)), v, device=0)
    c = bench.gen_queries(b, s, q, n, 7, torch.device("cuda", 0))
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(reps):
        t.predict_latency_many(c, out, stream=st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        t.predict_latency_many(c, out, stream=st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    import numpy as np
    from oracle.binding import or_interp3_many
    m = min(n, 2_000_000)
    want = or_interp3_many(t._b_axis, t._s_axis, t._q_axis, t.latency_ms, c[:m].cpu().numpy())
    same = np.array_equal(out[:m].cpu().numpy().view(np.int64), want.view(np.int64))
    print(f"parity vs oracle on {m} rows: {'OK' if same else 'MISMATCH'}")
    print(f"{n} queries: {ms:.3f} ms/launch, {n / ms / 1e6:.3f} e9 pred/s, "
          f"{32 * n / ms / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
