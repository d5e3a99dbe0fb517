"""BASELINE config 1 — the reference's own CPU-runnable case — end to end on the device:
the ResNet-50 table (b = 1..32 pow2, sm/quota 10..100) queried over the full sweep
b = 1..32 x sm = 10..100 x quota = 1..100 (291,200 points, most off-grid, q < 10 clamps),
latency and throughput bit-exact against the REFERENCE'S OWN compiled kernel
(oracle/_ref, built from hs/_kernels/_grid_cy.c) and most_efficient_config for 64 targets
log-spaced in [0.001, 2 x peak] at quota steps 1 and 10 against the C oracle."""

import numpy as np
import pytest

from oracle.binding import load_reference_kernel, or_most_efficient_config

from .conftest import same_bits

pytestmark = pytest.mark.gpu

BATCHES = [1, 2, 4, 8, 16, 32]


def resnet50_table():
    from paper_2505_01968_b200 import PerfTable
    s = list(range(10, 101, 10))
    q = list(range(10, 101, 10))
    # pkg/scripts/gen_tables.py:26-29 with the resnet50 parameters (8.0, 1.5, 0.35, 0.65)
    lat = np.array([[[(8.0 + 1.5 * b) * (0.35 + 0.65 * (100.0 / ss)) * (100.0 / qq)
                      for qq in q] for ss in s] for b in BATCHES])
    return PerfTable("resnet50", BATCHES, s, q, lat)


def sweep():
    b, s, q = np.meshgrid(np.arange(1, 33, dtype=np.float64),
                          np.arange(10, 101, dtype=np.float64),
                          np.arange(1, 101, dtype=np.float64), indexing="ij")
    return np.ascontiguousarray(np.column_stack([b.ravel(), s.ravel(), q.ravel()]))


def test_config1_sweep_matches_reference_kernel():
    ref = load_reference_kernel()
    if ref is None:
        pytest.skip("oracle/_ref not built (make -C oracle in the build container)")
    t = resnet50_table()
    c = sweep()
    assert len(c) == 291_200
    want = np.empty(len(c))
    ref.interp3_many(t._b_axis, t._s_axis, t._q_axis, t.latency_ms, c, want)
    import torch
    dc = torch.from_numpy(c).cuda()
    rps_d = torch.empty(len(c), dtype=torch.float64, device="cuda")
    lat = t.predict_latency_many(dc, rps_out=rps_d).cpu().numpy()
    rps = rps_d.cpu().numpy()
    assert same_bits(lat, want)
    assert same_bits(t.predict_latency_many(c), want)  # the host (pipelined) path too
    assert same_bits(rps, c[:, 0] / (want / 1000.0))  # throughput, hs/perf.py:95-98


def test_config1_search_64_targets_two_steps():
    from paper_2505_01968_b200 import PerfTableSet
    t = resnet50_table()
    peak = t.throughput(32, 100, 100)
    targets = np.geomspace(0.001, 2.0 * peak, 64).tolist()
    for step in (1, 10):
        ts = PerfTableSet([(t, None)] * len(targets), quota_step=step)
        got = ts.search(targets)
        for target, g in zip(targets, got):
            assert g == or_most_efficient_config(t._b_axis, t._s_axis, t._q_axis,
                                                 t.latency_ms, target, step, None)
        for target in targets[::9]:
            assert t.most_efficient_config(target, quota_step=step) == \
                or_most_efficient_config(t._b_axis, t._s_axis, t._q_axis, t.latency_ms,
                                         target, step, None)
