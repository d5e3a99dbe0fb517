"""Learned RaPP predictor (§8(f) row 4, parity unpinned: the reference has no learned
model).  The fused tcgen05 MLP kernel is checked against a PyTorch fp32 forward of the same
BF16-rounded weights and features; tolerance: relative error of the latency <= 2e-2 for
every row and median <= 2e-3 (the only differences are fp32 accumulation order and the
BF16 rounding of the hidden layer that order can flip)."""

import numpy as np
import pytest

from paper_2505_01968_b200 import learned


def test_zoo_graph_features():
    totals = {k: sum(o.flops for o in f()) for k, f in learned.ZOO.items()}
    # 2 x MACs per sample: ResNet-50 ~8.2 G, VGG-19 ~39 G, BERT-base(128) ~22 G,
    # MobileNetV2 ~0.6 G
    assert 7e9 < totals["resnet50"] < 9e9
    assert 3.5e10 < totals["vgg19"] < 4.2e10
    assert 1.8e10 < totals["bert-base"] < 2.6e10
    assert 4e8 < totals["mobilenet"] < 8e8
    feats = np.stack([learned.graph_features(f()) for f in learned.ZOO.values()])
    assert feats.shape == (4, learned.N_GRAPH) and np.all(np.isfinite(feats))
    assert np.allclose(feats[:, :8].sum(axis=1), 1.0, atol=1e-5)  # FLOP shares
    assert len({tuple(r) for r in feats.round(4)}) == 4             # distinct models


@pytest.mark.gpu
def test_mlp_kernel_matches_fp32_reference():
    lm = learned.LearnedPerfModel.zoo(seed=3)
    rng = np.random.default_rng(0)
    for model in range(len(lm.names)):
        n = 1000 + 37 * model  # ragged last tile
        c = np.column_stack([rng.uniform(0.5, 40, n), rng.uniform(0, 110, n),
                             rng.uniform(0, 110, n)])
        c[:50, 0] = rng.integers(1, 33, 50)
        got = lm.predict_many(model, c)
        want = lm.reference_forward(model, c)
        rel = np.abs(got - want) / np.abs(want)
        assert np.all(np.isfinite(got)) and np.all(got > 0)
        assert rel.max() <= 2e-2, (model, rel.max())
        assert np.median(rel) <= 2e-3, (model, np.median(rel))


@pytest.mark.gpu
def test_mlp_large_stream_and_perfmodel_view():
    import torch
    lm = learned.LearnedPerfModel.zoo(seed=1)
    n = 1 << 20
    g = torch.Generator(device="cuda").manual_seed(5)
    c = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    c[:, 0].uniform_(1, 32, generator=g)
    c[:, 1].uniform_(1, 100, generator=g)
    c[:, 2].uniform_(1, 100, generator=g)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    lm.predict_many_dev(2, c, out)
    idx = torch.randint(0, n, (4096,), device="cuda", generator=g)
    want = lm.reference_forward(2, c[idx].cpu().numpy())
    rel = np.abs(out[idx].cpu().numpy() - want) / want
    assert rel.max() <= 2e-2
    view = lm.for_model("bert-base")
    lat = view.predict_latency(8, 50, 50)
    assert lat > 0 and view.throughput(8, 50, 50) == pytest.approx(8 / (lat / 1000.0))


def _host_search(lm, model, target, bl, sl, step):
    """most_efficient_config (hs/perf.py:104-145) over the kernel's own predictions."""
    qs = list(range(step, 101, step))
    pts = np.array([(b, s, q) for s in sl for q in qs for b in bl], dtype=np.float64)
    lat = lm.predict_many(model, pts)
    rps = pts[:, 0] / (lat / 1000.0)
    best_meet, best_all = None, None
    for (b, s, q), r in zip(pts.astype(int).tolist(), rps.tolist()):
        ka = (-r, s * q, s, q, b)
        if best_all is None or ka < best_all:
            best_all = ka
        if r >= target:
            km = (s * q, s, q, b)
            if best_meet is None or km < best_meet:
                best_meet = km
    if best_meet is not None:
        return best_meet[3], best_meet[1], best_meet[2]
    return best_all[4], best_all[2], best_all[3]


@pytest.mark.gpu
def test_learned_search_matches_host_search_over_the_same_predictions():
    lm = learned.LearnedPerfModel.zoo(seed=2)
    bl, sl = [1, 2, 4, 8, 16, 32], list(range(5, 101, 5))
    rng = np.random.default_rng(9)
    models, targets = [], []
    for i in range(24):
        m = i % 4
        view = lm.for_model(lm.names[m])
        peak = view.throughput(32, 100, 100)
        targets.append(float(peak * rng.choice([1e-3, 0.05, 0.3, 0.7, 0.99, 5.0])))
        models.append(m)
    for step in (10, 25):
        got = lm.search(models, targets, batches=bl, sms=sl, quota_step=step)
        for m, t, g in zip(models, targets, got):
            assert g == _host_search(lm, m, t, bl, sl, step), (m, t, step)
