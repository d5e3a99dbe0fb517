"""The drop-in boundary binds the CALLER's types (CPU only): with the reference installed
(baseline/_ref) the records are hybridscale's own and every error derives from the
reference class of the same name, so the reference's `except` clauses catch them; with
RAPP_HOST_TYPES=standalone the package still imports and stands alone."""

import os
import subprocess
import sys

import pytest

from .conftest import REF_INSTALL, ROOT

hs = pytest.importorskip("hybridscale", reason="reference install baseline/_ref missing")


def test_records_are_the_references():
    from paper_2505_01968_b200 import core
    for name in ("ActionKind", "PodState", "ScalingAction", "ClusterState", "PodInstance",
                 "GpuDevice", "SmPartition", "FunctionSpec", "PodConfig"):
        assert getattr(core, name) is getattr(hs, name), name


def test_errors_derive_from_the_references():
    from hybridscale import errors as he

    from paper_2505_01968_b200 import errors as e
    assert e.BOUND
    for name in ("SchedulerError", "UnknownFunctionError", "UnknownPodError",
                 "UnknownGpuError", "PlacementError", "TableFormatError",
                 "FilterDegenerateError", "UnroutableFunctionError", "TraceFormatError",
                 "ConfigError", "InvariantViolation"):
        ours, theirs = getattr(e, name), getattr(he, name)
        assert issubclass(ours, theirs) and issubclass(ours, he.SchedulerError), name
        try:
            raise ours("x")
        except theirs:
            pass


def test_tick_emits_the_callers_types():
    from paper_2505_01968_b200 import core
    from paper_2505_01968_b200.tick import CallerTypes
    t = CallerTypes(hs.ClusterState())
    assert t.ScalingAction is hs.ScalingAction and t.kinds[2] is hs.ActionKind.HORIZONTAL_UP
    assert t.allocator is sys.modules["hybridscale.allocator"]
    assert CallerTypes(core.ClusterState()).ScalingAction is hs.ScalingAction


def test_standalone_mode():
    code = ("import sys; from paper_2505_01968_b200 import core, errors; "
            "from paper_2505_01968_b200.tick import CallerTypes; "
            "assert not errors.BOUND and 'hybridscale' not in sys.modules; "
            "t = CallerTypes(core.ClusterState()); assert t.allocator is None; "
            "assert t.ScalingAction is core.ScalingAction; "
            "assert issubclass(errors.TableFormatError, errors.SchedulerError); print('ok')")
    env = dict(os.environ, RAPP_HOST_TYPES="standalone",
               PYTHONPATH=os.pathsep.join([ROOT, REF_INSTALL]))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         cwd=ROOT, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr


def test_perf_reader_matches_reference_messages(tmp_path):
    """The csv-module reader (files outside the strict form) reports what the reference's
    reader reports (hs/perf.py:176-206), case by case."""
    from hybridscale import perf as hp

    from paper_2505_01968_b200 import perf as pp
    H = "function_id,batch,sm_percent,quota_percent,latency_ms\n"
    cases = {
        "empty": "",
        "bad_header": "a,b\n1,2\n",
        "only_header": H,
        "blank_and_quoted": H + "\n\"f\",1,50,10,\"2.5\"\n",
        "mixed": H + "f,1,50,10,2.0\ng,1,50,20,1.0\n f ,2,50,10,3.0\n",
        "dups": H + "f,1,50,10,2.0\nf,1,50,10,2.5\nf,1,50,20,1.0\n",
        "format": H + "f,1,50\nf,x,50,10,1.0\nf,1,50,10,nan\n,1,50,20,1.0\n",
        "empty_fid_first": H + ",1,50,10,2.0\nf,1,50,20,1.0\n",
    }
    for name, text in cases.items():
        path = tmp_path / f"{name}.csv"
        path.write_text(text, encoding="utf-8")
        fid, samples, issues = pp._read_samples(str(path))
        rfid, rsamples, rissues = hp._read_samples(str(path))
        assert fid == rfid, name
        assert repr(list(samples.items())) == repr(list(rsamples.items())), name
        assert [(i.kind, i.message, i.coord) for i in issues] == \
            [(i.kind, i.message, i.coord) for i in rissues], name


def test_new_pod_names_match_the_simulator_counter():
    """New pods are named pod-%06d from the simulator's counter (hs/sim.py:337-340); the
    tick names them from a table of three-digit suffixes, across the 999/1000 and
    999,999/1,000,000 boundaries too."""
    from paper_2505_01968_b200.tick import _pod_names
    for c0, n in [(0, 0), (0, 5), (995, 10), (123_456, 300), (999_995, 10), (1_234_560, 2_500)]:
        assert _pod_names(c0, n) == ["pod-%06d" % c for c in range(c0, c0 + n)]


def test_new_pod_name_cache_follows_the_counter():
    """TickEngine's name cache (topped up between rapp_tick_submit and rapp_tick_collect)
    hands out exactly the pod-%06d names of the counter values a tick consumes, including
    ticks that outrun the cache and counters that jump outside it."""
    from paper_2505_01968_b200.tick import TickEngine

    class Stub:
        counter = 0
        _NAMES_TOPUP_MAX = 1024
        _top_up_names = TickEngine._top_up_names
        _new_names = TickEngine._new_names

    e = Stub()
    import numpy as np
    rng = np.random.default_rng(3)
    for step in range(200):
        e._top_up_names()
        k = int(rng.choice([0, 1, 5, 300, 700, 2500]))
        if step == 120:
            e.counter += 10_000  # e.g. a rebuilt engine: the cache restarts
            e._top_up_names()
        got = e._new_names(e.counter, k)
        assert got == ["pod-%06d" % c for c in range(e.counter, e.counter + k)]
        e.counter += k


def test_pod_id_mirror_and_lazy_views():
    """TickEngine's object-array mirror of the pod id list (for gathering a tick's pod ids
    by device pod index) follows the list as ticks append to it, across capacity growth,
    and the lazily named function ids of new pods come out in pod order."""
    import numpy as np
    from paper_2505_01968_b200.tick import TickEngine

    class Stub:
        _ids_mirror = TickEngine._ids_mirror
        pod_fids = TickEngine.pod_fids

    e = Stub()
    e.pod_ids = [f"init-{i}" for i in range(5)]
    e.fids = ["fa", "fb", "fc"]
    e._fids_np = np.array(e.fids, dtype=object)
    e._pod_fids = ["fa"] * 5
    e._pod_fn_pending = []
    rng = np.random.default_rng(7)
    want_f = list(e._pod_fids)
    for _ in range(40):
        k = int(rng.integers(0, 900))
        e.pod_ids.extend(f"pod-{len(e.pod_ids) + j:06d}" for j in range(k))
        fn = rng.integers(0, 3, k).astype(np.int32)
        e._pod_fn_pending.append(fn)
        want_f.extend(e.fids[i] for i in fn)
        idx = rng.integers(0, len(e.pod_ids), 50)
        assert e._ids_mirror()[idx].tolist() == [e.pod_ids[i] for i in idx]
    assert e.pod_fids == want_f
