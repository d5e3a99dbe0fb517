"""The CPU oracle (oracle/) pinned against the reference's golden vectors (CPU only)."""

import math

import numpy as np
import pytest

from oracle.binding import (load_reference_kernel, or_interp3_many, or_locate,
                            or_most_efficient_config)

from .conftest import fromhex, golden_table_arrays, same_bits


def test_oracle_interp_matches_golden(interp_golden):
    for rec in interp_golden["tables"]:
        b, s, q, v = golden_table_arrays(rec["table"])
        coords = fromhex(rec["coords"]).reshape(-1, 3)
        want = fromhex(rec["latency"])
        got = or_interp3_many(b, s, q, v, coords)
        assert same_bits(got, want), rec["table"]["function_id"]


def test_oracle_locate_matches_golden(interp_golden):
    for rec in interp_golden["locate"]:
        axis = fromhex(rec["axis"])
        lo, hi, t = or_locate(axis, float.fromhex(rec["x"]))
        want_t = float.fromhex(rec["t"])
        assert (lo, hi) == (rec["lo"], rec["hi"])
        assert (math.isnan(t) and math.isnan(want_t)) or t == want_t


def test_oracle_search_matches_golden(mec_golden):
    tables = {t["function_id"]: golden_table_arrays(t) for t in mec_golden["tables"]}
    for case in mec_golden["cases"]:
        b, s, q, v = tables[case["table"]]
        got = or_most_efficient_config(b, s, q, v, float.fromhex(case["target"]),
                                       case["step"], case["batches"])
        assert list(got) == case["result"], case


def test_oracle_search_rejects_bad_inputs(mec_golden):
    b, s, q, v = golden_table_arrays(mec_golden["tables"][0])
    with pytest.raises(ValueError):
        or_most_efficient_config(b, s, q, v, 0.0, 10)
    with pytest.raises(ValueError):
        or_most_efficient_config(b, s, q, v, 1.0, 0)


def test_oracle_matches_reference_build_on_random_inputs():
    """oracle/_ref is the reference's own compiled _grid_cy (built from /root/reference)."""
    ref = load_reference_kernel()
    if ref is None:
        pytest.skip("oracle/_ref not built (reference tree absent)")
    rng = np.random.default_rng(7)
    b = np.array([1.0, 2.0, 4.0, 8.0, 16.0, 32.0])
    s = np.arange(10.0, 101.0, 10.0)
    q = np.arange(10.0, 101.0, 10.0)
    v = np.ascontiguousarray(rng.uniform(1, 100, (6, 10, 10)))
    coords = np.column_stack([rng.uniform(0, 40, 50000), rng.uniform(0, 110, 50000),
                              rng.uniform(0, 110, 50000)])
    coords[::3] = np.round(coords[::3])
    want = np.empty(len(coords))
    ref.interp3_many(b, s, q, v, coords, want)
    assert same_bits(or_interp3_many(b, s, q, v, coords), want)
