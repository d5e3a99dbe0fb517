#!/usr/bin/env python3
"""Generates the golden vectors in tests/golden/ by running the REAL reference.

Run in the build container only (the reference tree is absent on the GPU box):

    python tests/golden/gen_golden.py            # all sets
    python tests/golden/gen_golden.py interp mec # selected sets

The reference package is imported from a scratch copy (/tmp/refpkg) whose
Cython kernel is built in place, because /root/reference is read-only.
Doubles are stored as float.hex() strings so comparisons are 0-ulp.
"""

from __future__ import annotations

import json
import os
import random
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg"
SCRATCH = "/tmp/refpkg"


def import_reference():
    if not os.path.exists(os.path.join(SCRATCH, "src", "hybridscale")):
        shutil.copytree(REF_PKG, SCRATCH)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                       check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    sys.path.insert(0, SCRATCH)  # for `tests.conftest` / `tests.oracles`
    import hybridscale
    assert hybridscale.KERNEL_BACKEND == "cython", hybridscale.KERNEL_BACKEND
    return hybridscale


def hx(x: float) -> str:
    return float(x).hex()


def hx_arr(a) -> list[str]:
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def table_dict(t) -> dict:
    return {"function_id": t.function_id, "batches": list(t.batches), "sms": list(t.sms),
            "quotas": list(t.quotas), "latency_ms": hx_arr(t.latency_ms)}


def dump(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


# -- interpolation ------------------------------------------------------------


def gen_interp(hs):
    from hybridscale import load_table
    from hybridscale._kernels import _grid_cy, locate
    tables = [load_table(os.path.join(REF_PKG, "tables", n))
              for n in ("resnet50.csv", "bert-small.csv")]
    # the test_kernels.py:_grid() table (pkg/tests/test_kernels.py:12-19)
    from tests.test_kernels import _grid
    b, s, q, v = _grid()
    grid_tab = hs.PerfTable("kernels-grid", [1, 2, 4, 8], [25, 50, 75, 100],
                            [10, 40, 70, 100], v)
    tables.append(grid_tab)
    rng = np.random.default_rng(20261017)
    out = {"tables": [], "locate": []}
    for t in tables:
        n = 3000
        c = np.column_stack([
            rng.uniform(t.batches[0] - 1, t.batches[-1] + 1, n),
            rng.uniform(t.sms[0] - 10, t.sms[-1] + 10, n),
            rng.uniform(t.quotas[0] - 10, t.quotas[-1] + 10, n)])
        # exact node hits, clamps, integers and specials
        c[0::9, 0] = rng.choice(t.batches, len(c[0::9]))
        c[1::9, 1] = rng.choice(t.sms, len(c[1::9]))
        c[2::9, 2] = rng.choice(t.quotas, len(c[2::9]))
        c[3::11] = np.round(c[3::11])
        c[5] = [np.nan, 50.0, 50.0]
        c[6] = [2.0, np.nan, 50.0]
        c[7] = [2.0, 50.0, np.nan]
        c[8] = [np.inf, -np.inf, 1e308]
        c[9] = [-0.0, 0.0, -1e-300]
        res = np.empty(n)
        _grid_cy.interp3_many(t._b_axis, t._s_axis, t._q_axis, t.latency_ms, c, res)
        out["tables"].append({"table": table_dict(t), "coords": hx_arr(c),
                              "latency": hx_arr(res)})
    axis = np.array([10.0, 20.0, 40.0])
    for x in [10.0, 20.0, 40.0, 25.0, 5.0, 99.0, 39.999999, 10.000001, float("nan"),
              float("inf"), float("-inf"), -0.0]:
        lo, hi, t = locate(axis, x)
        out["locate"].append({"axis": hx_arr(axis), "x": hx(x), "lo": lo, "hi": hi,
                              "t": hx(t)})
    one = np.array([7.0])
    for x in [7.0, 1.0, 9.0, float("nan")]:
        lo, hi, t = locate(one, x)
        out["locate"].append({"axis": hx_arr(one), "x": hx(x), "lo": lo, "hi": hi,
                              "t": hx(t)})
    dump("interp.json", out)


# -- most_efficient_config ------------------------------------------------------


def gen_mec(hs):
    from hybridscale import load_table
    from tests.conftest import make_conformance_table, random_monotone_table
    tables = [load_table(os.path.join(REF_PKG, "tables", n))
              for n in ("resnet50.csv", "bert-small.csv")]
    tables.append(make_conformance_table())
    rng = random.Random(4242)
    for i in range(12):
        tables.append(random_monotone_table(rng, rng.randint(1, 5), rng.randint(1, 5),
                                            rng.randint(1, 6), function_id=f"rand-{i}"))
    cases = []
    for t in tables:
        peak = t.throughput(t.batches[-1], t.sms[-1], 100)
        targets = [0.001, 0.1 * peak, 0.3 * peak, 0.5 * peak, 0.75 * peak, 0.99 * peak,
                   peak, 2.0 * peak, 1e9]
        # tie edge: targets exactly equal to a lattice throughput
        for _ in range(4):
            b = rng.choice(t.batches)
            s = rng.choice(t.sms)
            qq = rng.choice(range(10, 101, 10))
            targets.append(t.throughput(b, s, qq))
        for step in (1, 7, 10, 20, 25, 50, 100):
            for batches in (None, t.batches[:1], [3, 5], [0, 1000], [t.batches[-1], 1]):
                for target in targets:
                    got = t.most_efficient_config(target, quota_step=step, batches=batches)
                    cases.append({"table": t.function_id, "target": hx(target),
                                  "step": step, "batches": batches, "result": list(got)})
    dump("mec.json", {"tables": [table_dict(t) for t in tables], "cases": cases})


GENERATORS = {"interp": gen_interp, "mec": gen_mec}


def main(argv):
    hs = import_reference()
    names = argv or list(GENERATORS)
    for name in names:
        GENERATORS[name](hs)


if __name__ == "__main__":
    main(sys.argv[1:])
