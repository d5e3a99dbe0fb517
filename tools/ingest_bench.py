"""Times load_table on config-2-sized tables (6 x 100 x 100 = 60,000 rows each).

    python tools/ingest_bench.py [n_tables]            # this package (GPU)
    python tools/ingest_bench.py [n_tables] --reference  # the reference (build container)"""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main(n=8, reference=False):
    if reference:
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                        "tests", "golden"))
        import gen_golden
        hs = gen_golden.import_reference()
        load_table, save_table, PerfTable = hs.load_table, hs.save_table, hs.PerfTable
    else:
        from paper_2505_01968_b200 import PerfTable, load_table, save_table
    tmp = tempfile.mkdtemp()
    paths = []
    for i, (name, b, s, q, v) in enumerate((bench.config2_arrays() * 4)[:n]):
        t = PerfTable(f"{name}-{i}", bench.BATCHES, list(range(1, 101)), list(range(1, 101)), v)
        p = os.path.join(tmp, f"t{i}.csv")
        save_table(t, p)
        paths.append(p)
    load_table(paths[0])  # warm-up (library / context / CUDA init)
    t0 = time.perf_counter()
    for p in paths:
        load_table(p)
    dt = (time.perf_counter() - t0) / len(paths)
    print(f"{'reference' if reference else 'b200'} load_table: {dt * 1e3:.2f} ms per "
          f"60,000-row table ({len(paths)} tables)")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 8,
         "--reference" in sys.argv)
