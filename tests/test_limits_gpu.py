"""Error paths of the device layouts' hard limits (the reference has none of these; the B200
path refuses loudly instead of truncating or overflowing):

* the tick world holds at most 128 pods per managed function (rapp_tick.cu kMaxPods) — at
  upload and when a tick would create the 129th;
* pod ids are at most 32 UTF-8 bytes (the device compares them as packed big-endian bytes);
* the lattice search packs (s*q, s index, q, b index) into 64 bits: at most 4,096 sm nodes
  and 4,096 batch-lattice entries, integral sm values below 2^24."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

QUOTAS = list(range(10, 101, 10))


def _table(fid="conf-fn", batches=(8,), sms=(25, 50), quotas=QUOTAS):
    from paper_2505_01968_b200 import PerfTable
    b = np.asarray(batches, float)[:, None, None]
    s = np.asarray(sms, float)[None, :, None]
    q = np.asarray(quotas, float)[None, None, :]
    lat = (4.0 + b) * (0.3 + 0.7 * 100.0 / s) * (100.0 / q)
    return PerfTable(fid, list(batches), list(sms), list(quotas), lat)


def _world(npods, ngpus, pid=lambda i: f"p{i:04d}", sm=10, q=10):
    from bench import place_initial
    from paper_2505_01968_b200.core import (ClusterState, FunctionSpec, GpuDevice, PodConfig,
                                            PodInstance, PodState)
    c = ClusterState(gpus={f"gpu-{i:03d}": GpuDevice(f"gpu-{i:03d}") for i in range(ngpus)})
    for i in range(npods):
        g = f"gpu-{i // 10:03d}"  # 10 pods of 10% SM x 10% quota per GPU
        place_initial(c, PodInstance(pid(i), "conf-fn", 8, sm, q, g, state=PodState.RUNNING), g)
    fn = FunctionSpec("conf-fn", 20.0, perf_table_ref="conf-fn", allowed_batches=[8],
                      initial=PodConfig(8, sm, q))
    return fn, c


def _engine(fn, cluster, tables, policy="hybrid"):
    from paper_2505_01968_b200.autoscaler import ScalerConfig
    from paper_2505_01968_b200.tick import TickEngine
    return TickEngine([fn], tables, cluster, ScalerConfig(alpha=0.9, beta=0.5, delta_iq=10),
                      pod_counter=len(cluster.pods), policy=policy)


def test_tick_world_rejects_more_than_128_pods_per_function():
    from paper_2505_01968_b200.errors import DeviceError
    tables = {"conf-fn": _table(sms=(10, 50, 100))}
    fn, c = _world(128, 20)
    eng = _engine(fn, c, tables)  # 128 pods: accepted
    eng.close()
    fn, c = _world(129, 20)
    with pytest.raises(DeviceError, match="more than 128 pods"):
        _engine(fn, c, tables)


def test_tick_refuses_to_create_the_129th_pod():
    """A replica scale-up past the per-function pod capacity fails the tick with the
    device's error instead of writing past the function's pod list."""
    from paper_2505_01968_b200.errors import DeviceError
    tables = {"conf-fn": _table(sms=(10, 50, 100))}
    fn, c = _world(126, 40)
    eng = _engine(fn, c, tables, policy="horizontal-only")
    with pytest.raises(DeviceError):
        eng.tick(2000.0, {"conf-fn": 10_000_000})  # wants far more than 2 new replicas
    eng.close()


def test_pod_ids_longer_than_32_bytes_are_rejected():
    from paper_2505_01968_b200.errors import ConfigError
    tables = {"conf-fn": _table(sms=(10, 50, 100))}
    fn, c = _world(2, 1, pid=lambda i: f"{'x' * 31}{i}")  # 32 bytes: fine
    _engine(fn, c, tables).close()
    fn, c = _world(2, 1, pid=lambda i: f"{'x' * 32}{i}")  # 33 bytes
    with pytest.raises(ConfigError, match="at most 32 UTF-8 bytes"):
        _engine(fn, c, tables)
    fn, c = _world(2, 1, pid=lambda i: f"p\x00{i}")
    with pytest.raises(ConfigError):
        _engine(fn, c, tables)


def test_lattice_search_key_limits():
    from paper_2505_01968_b200 import PerfTableSet
    from paper_2505_01968_b200.errors import DeviceError
    ok = _table(sms=list(range(1, 4097)), quotas=[50, 100])  # 4,096 sm nodes: the maximum
    s = PerfTableSet([(ok, [8])], quota_step=50)
    assert len(s.search(np.array([1.0]))) == 1
    s.close()
    wide = _table(sms=list(range(1, 4098)), quotas=[50, 100])
    with pytest.raises(DeviceError, match="outside \\[1, 4096\\]"):
        PerfTableSet([(wide, [8])], quota_step=50)
    tall = _table(batches=list(range(1, 4098)), sms=[50, 100], quotas=[50, 100])
    with pytest.raises(DeviceError, match="outside \\[1, 4096\\]"):
        PerfTableSet([(tall, list(range(1, 4098)))], quota_step=50)
    huge = _table(sms=[50, 1 << 24], quotas=[50, 100])  # s*q would overflow the cost field
    with pytest.raises(DeviceError, match="2\\^24"):
        PerfTableSet([(huge, [8])], quota_step=50)


def test_tick_world_size_limits_at_the_c_abi():
    """rapp_tick_create refuses worlds beyond its index widths (2^18 GPUs: the rank field of
    the packed argmin keys; 2^20 functions) before touching any input array."""
    import ctypes
    from paper_2505_01968_b200 import _lib
    from paper_2505_01968_b200.errors import DeviceError
    from paper_2505_01968_b200.tick import ScalerConfigC
    lib = _lib.load()
    ctx = _lib.Context.get(0)
    cfg = ScalerConfigC(0.9, 0.5, 1000.0, 1.0, 10, 0, 2.0, 5000.0, 1.0, 4.0, 1.0, 16.0, 1.0,
                        0, 0)
    h = _lib.c_vp()
    for n_fns, n_gpus in (((1 << 20) + 1, 1), (1, (1 << 18) + 1)):
        rc = lib.rapp_tick_create(ctx.handle, ctypes.byref(cfg), n_fns, None, None, n_gpus,
                                  None, None, None, 0, None, 0, ctypes.byref(h))
        with pytest.raises(DeviceError, match="exceeds the tick's limits"):
            _lib.check(rc, "TickEngine")


def test_tick_submit_collect_pairing():
    """rapp_tick_submit / rapp_tick_collect (the two halves of rapp_tick_run) refuse an
    unpaired collect, a second submit and any other world call in between, and a paired
    call returns what rapp_tick_run returns."""
    import ctypes
    from paper_2505_01968_b200 import _lib
    tables = {"conf-fn": _table(sms=(10, 50, 100))}
    fn, c = _world(4, 4)
    eng = _engine(fn, c, tables)
    lib = _lib.load()
    n = ctypes.c_int64()
    arr = np.array([50], dtype=np.int64)
    assert lib.rapp_tick_collect(eng._h, eng._act_addr, len(eng._act_buf), ctypes.byref(n),
                                 None, None) == _lib.RAPP_E_ARG
    assert "no submitted tick" in _lib.last_error()
    assert lib.rapp_tick_submit(eng._h, 1000.0, arr.ctypes.data, None, None,
                                len(eng._act_buf)) == 0
    assert lib.rapp_tick_submit(eng._h, 1000.0, arr.ctypes.data, None, None,
                                len(eng._act_buf)) == _lib.RAPP_E_ARG
    pods = np.array([0], dtype=np.int64)
    assert lib.rapp_tick_release(eng._h, pods.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                 1) == _lib.RAPP_E_ARG
    assert lib.rapp_tick_collect(eng._h, eng._act_addr, len(eng._act_buf), ctypes.byref(n),
                                 None, None) == 0
    eng._bookkeep(eng._act_buf[:n.value].copy())  # keep the host's pod list in step
    # the engine goes on normally afterwards (its own tick is submit + collect)
    res = eng.tick(2000.0, {"conf-fn": 50})
    assert res.observed["conf-fn"] >= 0.0
    eng.close()
