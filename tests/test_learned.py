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
