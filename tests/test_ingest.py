"""Perf-table ingest (hs/perf.py:155-267): the native strict-form CSV reader (CPU) and the
device grid assembly + validation (GPU), against reports and tables the REAL reference
produced for the same files (tests/golden/ingest.json, gen_golden.py:gen_ingest)."""

import csv
import ctypes
import io
import os

import numpy as np
import pytest

from paper_2505_01968_b200 import _lib

from .conftest import fromhex, load_golden, same_bits

STRICT = {"ref_resnet50.csv", "ref_bert-small.csv", "valid", "valid_shuffled", "valid_crlf",
          "valid_float_forms", "valid_no_trailing_newline", "valid_single_cell", "valid_flat",
          "duplicate", "duplicate_shuffled", "missing", "missing_and_bad", "non_positive",
          "mono_batch", "mono_sm", "mono_quota", "many_issues", "negative_axes",
          "big_batch_values"}


@pytest.fixture(scope="module")
def golden():
    return load_golden("ingest.json")


def native_parse(body: bytes):
    lib = _lib.load()
    cap = body.count(b"\n") + 1
    b, s, q = (np.empty(cap, dtype=np.int64) for _ in range(3))
    lat = np.empty(cap, dtype=np.float64)
    n, reg = ctypes.c_int64(), ctypes.c_int32()
    fid = ctypes.create_string_buffer(256)
    _lib.check(lib.rapp_csv_parse(body, len(body), cap, _lib.i64ptr(b), _lib.i64ptr(s),
                                  _lib.i64ptr(q), _lib.dptr(lat), ctypes.byref(n), fid, 256,
                                  ctypes.byref(reg)))
    k = n.value
    return bool(reg.value), fid.value.decode(), b[:k], s[:k], q[:k], lat[:k]


def test_native_reader_accepts_exactly_the_strict_form(golden):
    for name, rec in golden.items():
        regular = native_parse(rec["csv"].encode())[0]
        assert regular == (name in STRICT), name


def test_native_reader_rows_equal_the_csv_module(golden):
    for name in STRICT:
        body = golden[name]["csv"]
        _, fid, b, s, q, lat = native_parse(body.encode())
        rows = [r for r in csv.reader(io.StringIO(body, newline=""))][1:]
        rows = [r for r in rows if r]
        assert fid == rows[0][0].strip()
        assert b.tolist() == [int(r[1]) for r in rows]
        assert s.tolist() == [int(r[2]) for r in rows]
        assert q.tolist() == [int(r[3]) for r in rows]
        assert same_bits(lat, np.array([float(r[4]) for r in rows])), name


def test_native_reader_literals_round_trip():
    rng = np.random.default_rng(3)
    vals = np.concatenate([rng.uniform(0, 1e3, 2000), 10.0 ** rng.uniform(-300, 300, 2000),
                           [5e-324, 1.7976931348623157e308, 0.1, 1 / 3]])
    lines = ["function_id,batch,sm_percent,quota_percent,latency_ms"]
    lines += [f"f,{i},1,1,{float(v)!r}" for i, v in enumerate(vals)]
    lines += [f"f,{len(vals) + i},1,1,{v:.17e}" for i, v in enumerate(vals)]
    reg, _, _, _, _, lat = native_parse(("\n".join(lines) + "\n").encode())
    assert reg
    want = np.concatenate([vals, [float(f"{v:.17e}") for v in vals]])
    assert same_bits(lat, want)


def _write(tmp_path, body):
    p = tmp_path / "table.csv"
    p.write_bytes(body.encode("utf-8"))
    return str(p)


@pytest.mark.gpu
def test_validate_table_file_matches_reference(tmp_path, golden):
    from paper_2505_01968_b200 import validate_table_file
    for name, rec in golden.items():
        rep = validate_table_file(_write(tmp_path, rec["csv"]))
        want = rec["report"]
        assert rep.function_id == want["function_id"], name
        assert (rep.batches, rep.sms, rep.quotas) == \
            (want["batches"], want["sms"], want["quotas"]), name
        got = [[i.kind, i.message, list(i.coord) if i.coord else None] for i in rep.issues]
        assert got == want["issues"], name


@pytest.mark.gpu
def test_load_table_matches_reference(tmp_path, golden):
    from paper_2505_01968_b200 import load_table
    from paper_2505_01968_b200.errors import TableFormatError
    for name, rec in golden.items():
        path = _write(tmp_path, rec["csv"])
        if rec["load"]["ok"]:
            t = load_table(path)
            w = rec["load"]["table"]
            assert t.function_id == w["function_id"], name
            assert (t.batches, t.sms, t.quotas) == (w["batches"], w["sms"], w["quotas"]), name
            assert same_bits(t.latency_ms.ravel(), fromhex(w["latency_ms"])), name
        else:
            with pytest.raises(TableFormatError) as ei:
                load_table(path)
            assert str(ei.value) == f"{path}: {rec['load']['message']}", name


@pytest.mark.gpu
def test_fine_grid_round_trip_and_prediction(tmp_path):
    """A config-2 table (6 x 100 x 100 = 60,000 rows) through save_table -> load_table,
    then predictions from the loaded table equal predictions from the original."""
    import bench
    from paper_2505_01968_b200 import PerfTable, load_table, save_table
    _, b, s, q, v = bench.config2_arrays()[1]
    t = PerfTable("vgg19", bench.BATCHES, list(range(1, 101)), list(range(1, 101)), v)
    path = str(tmp_path / "vgg19.csv")
    save_table(t, path)
    u = load_table(path)
    assert (u.batches, u.sms, u.quotas) == (t.batches, t.sms, t.quotas)
    assert same_bits(u.latency_ms, t.latency_ms)
    rng = np.random.default_rng(1)
    c = np.column_stack([rng.uniform(1, 32, 5000), rng.uniform(1, 100, 5000),
                         rng.uniform(1, 100, 5000)])
    assert same_bits(u.predict_latency_many(c), t.predict_latency_many(c))


@pytest.mark.gpu
def test_ingest_duplicates_in_row_order(tmp_path):
    """Strict-form file with many repeated coordinates: duplicates are found on the device
    and reported in row order, the first one raised by load_table."""
    from paper_2505_01968_b200 import load_table, validate_table_file
    from paper_2505_01968_b200.errors import TableFormatError
    rng = np.random.default_rng(5)
    rows = [(b, s, q) for b in (1, 2, 4) for s in range(10, 101, 10) for q in range(10, 101, 10)]
    extra = [rows[i] for i in rng.integers(0, len(rows), 50)]
    allrows = rows + extra
    lines = ["function_id,batch,sm_percent,quota_percent,latency_ms"]
    lines += [f"f,{b},{s},{q},{1000.0 / s / q * b!r}" for b, s, q in allrows]
    path = _write(tmp_path, "\n".join(lines) + "\n")
    seen, want = set(), []
    for c in allrows:
        if c in seen:
            want.append(f"duplicate sample at batch={c[0]} sm={c[1]} quota={c[2]}")
        seen.add(c)
    rep = validate_table_file(path)
    assert [i.message for i in rep.issues] == want
    with pytest.raises(TableFormatError, match=want[0]):
        load_table(path)
