import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
# the reference package is the drop-in's caller: its install (baseline/_ref, git-ignored,
# travels to the GPU box) makes the B200 path bind the caller's record and error types
REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(os.path.join(REF_INSTALL, "hybridscale")) and REF_INSTALL not in sys.path:
    sys.path.append(REF_INSTALL)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and librapp_b200.so")


def fromhex(xs):
    return np.array([float.fromhex(x) for x in xs], dtype=np.float64)


def load_golden(name):
    with open(os.path.join(GOLDEN, name), encoding="utf-8") as fh:
        return json.load(fh)


def golden_table_arrays(t):
    """(b_axis, s_axis, q_axis, values) float64 arrays of a golden table record."""
    b = np.asarray(t["batches"], dtype=np.float64)
    s = np.asarray(t["sms"], dtype=np.float64)
    q = np.asarray(t["quotas"], dtype=np.float64)
    v = fromhex(t["latency_ms"]).reshape(len(b), len(s), len(q))
    return b, s, q, v


def same_bits(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and bool(np.all(a.view(np.int64) == b.view(np.int64)))


@pytest.fixture(scope="session")
def interp_golden():
    return load_golden("interp.json")


@pytest.fixture(scope="session")
def mec_golden():
    return load_golden("mec.json")
