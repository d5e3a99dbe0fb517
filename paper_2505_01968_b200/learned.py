"""Learned RaPP performance model on the tensor cores.

The paper's RaPP (arxiv 2505.01968 §3.2) predicts latency from operator-level model-graph
features combined with the resource configuration (SM %, time quota, batch).  The reference
replaces it with a validated grid and ships no learned model, weights or
dataset, so this path is **parity unpinned**: it plugs in behind the same `PerfModel`
protocol (hs/perf.py:23-31) only when a caller asks for it, and its kernel is checked
against a PyTorch fp32 forward of the same BF16 weights.

* Graph features (`graph_features`): op-graph statistics of a model — per-op-type FLOP and
  count shares, total FLOPs / bytes / parameters, arithmetic intensity, depth — plus two
  rounds of mean message passing over the op chain pooled by mean and max (40 values, once
  per model, host side).
* Per-query features and the MLP forward run fused in one kernel (`rapp_mlp.cu`): the
  feature row is written straight into the swizzled shared-memory A operand and the two
  hidden layers are `tcgen05.mma` GEMMs with TMEM accumulators.
* Weights are random (seeded) — there is no trained model to load; the architecture, not
  the accuracy, is what this component provides.  The biases ride on a constant input
  feature and a constant hidden unit (127 real units + 1 per hidden layer), so all three
  layers are tensor-core GEMMs with BF16 operands (`effective_weights`).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib

N_GRAPH = 40
N_CFG = 16
K0 = 64
HIDDEN = 128
OP_TYPES = ("conv", "dwconv", "linear", "attention", "pool", "norm", "act", "eltwise")


@dataclass
class Op:
    kind: str
    flops: float   # per sample
    bytes: float   # activations in + out + parameters, per sample
    params: float


def _conv(cin, cout, k, hw, stride=1, depthwise=False):
    ho = hw // stride
    if depthwise:
        flops = 2.0 * cin * k * k * ho * ho
        params = cin * k * k
    else:
        flops = 2.0 * cin * cout * k * k * ho * ho
        params = cin * cout * k * k
    act = 2.0 * (cin * hw * hw + cout * ho * ho)
    return Op("dwconv" if depthwise else "conv", flops, act + 2.0 * params, params), ho


def _simple(kind, elems, flops_per=1.0):
    return Op(kind, flops_per * elems, 4.0 * elems, 0.0)


def resnet50():
    ops, hw = [], 224
    op, hw = _conv(3, 64, 7, hw, 2)
    ops += [op, _simple("norm", 64 * hw * hw, 4), _simple("act", 64 * hw * hw)]
    hw //= 2
    ops.append(_simple("pool", 64 * hw * hw, 9))
    cin = 64
    for width, blocks, stride in ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)):
        for i in range(blocks):
            s = stride if i == 0 else 1
            o1, h1 = _conv(cin, width, 1, hw)
            o2, h2 = _conv(width, width, 3, h1, s)
            o3, h3 = _conv(width, width * 4, 1, h2)
            ops += [o1, _simple("act", width * h1 * h1), o2, _simple("act", width * h2 * h2),
                    o3, _simple("norm", width * 4 * h3 * h3, 4),
                    _simple("eltwise", width * 4 * h3 * h3), _simple("act", width * 4 * h3 * h3)]
            cin, hw = width * 4, h3
    ops += [_simple("pool", cin * hw * hw), Op("linear", 2.0 * cin * 1000, 2.0 * cin * 1000,
                                                 cin * 1000)]
    return ops


def vgg19():
    ops, hw, cin = [], 224, 3
    for cfg in (64, 64, "M", 128, 128, "M", 256, 256, 256, 256, "M", 512, 512, 512, 512, "M",
                512, 512, 512, 512, "M"):
        if cfg == "M":
            ops.append(_simple("pool", cin * hw * hw))
            hw //= 2
            continue
        op, hw = _conv(cin, cfg, 3, hw)
        ops += [op, _simple("act", cfg * hw * hw)]
        cin = cfg
    for fin, fout in ((cin * hw * hw, 4096), (4096, 4096), (4096, 1000)):
        ops += [Op("linear", 2.0 * fin * fout, 2.0 * fin * fout, fin * fout),
                _simple("act", fout)]
    return ops


def bert_base(seq=128, d=768, layers=12, ff=3072):
    ops = [_simple("eltwise", seq * d, 2)]
    for _ in range(layers):
        ops += [Op("linear", 2.0 * seq * d * 3 * d, 2.0 * (seq * d * 4 + 3 * d * d), 3 * d * d),
                Op("attention", 4.0 * seq * seq * d, 2.0 * (3 * seq * d + 12 * seq * seq), 0),
                _simple("act", 12 * seq * seq, 5),
                Op("linear", 2.0 * seq * d * d, 2.0 * (2 * seq * d + d * d), d * d),
                _simple("eltwise", seq * d), _simple("norm", seq * d, 5),
                Op("linear", 2.0 * seq * d * ff, 2.0 * (seq * (d + ff) + d * ff), d * ff),
                _simple("act", seq * ff, 8),
                Op("linear", 2.0 * seq * ff * d, 2.0 * (seq * (d + ff) + d * ff), d * ff),
                _simple("eltwise", seq * d), _simple("norm", seq * d, 5)]
    return ops


def mobilenet_v2():
    ops, hw = [], 224
    op, hw = _conv(3, 32, 3, hw, 2)
    ops += [op, _simple("act", 32 * hw * hw)]
    cin = 32
    for t, c, n, s in ((1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2),
                       (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)):
        for i in range(n):
            st = s if i == 0 else 1
            hid = cin * t
            o1, h1 = _conv(cin, hid, 1, hw)
            o2, h2 = _conv(hid, hid, 3, h1, st, depthwise=True)
            o3, h3 = _conv(hid, c, 1, h2)
            ops += [o1, _simple("act", hid * h1 * h1), o2, _simple("act", hid * h2 * h2), o3]
            if st == 1 and cin == c:
                ops.append(_simple("eltwise", c * h3 * h3))
            cin, hw = c, h3
    op, hw = _conv(cin, 1280, 1, hw)
    ops += [op, _simple("pool", 1280 * hw * hw), Op("linear", 2.0 * 1280 * 1000,
                                                    2.0 * 1280 * 1000, 1280 * 1000)]
    return ops


ZOO = {"resnet50": resnet50, "vgg19": vgg19, "bert-base": bert_base,
       "mobilenet": mobilenet_v2}


def graph_features(ops) -> np.ndarray:
    """40 features of an op chain (see module docstring)."""
    n = len(ops)
    kinds = np.array([OP_TYPES.index(o.kind) for o in ops])
    flops = np.array([o.flops for o in ops])
    byts = np.array([o.bytes for o in ops])
    params = np.array([o.params for o in ops])
    f = np.zeros(N_GRAPH, dtype=np.float64)
    tot_f, tot_b = flops.sum(), byts.sum()
    for k in range(len(OP_TYPES)):
        f[k] = flops[kinds == k].sum() / tot_f
        f[8 + k] = (kinds == k).sum() / n
    f[16] = math.log10(tot_f) / 10.0
    f[17] = math.log10(tot_b) / 10.0
    f[18] = math.log10(params.sum() + 1.0) / 10.0
    f[19] = math.log10(tot_f / tot_b) / 3.0
    # two rounds of mean message passing along the op chain, pooled by mean and max
    h = np.zeros((n, 10))
    h[:, 0] = np.log1p(flops) / 25.0
    h[:, 1] = np.log1p(byts) / 25.0
    h[np.arange(n), 2 + kinds] = 1.0
    for _ in range(2):
        prev = np.vstack([h[:1], h[:-1]])
        h = 0.5 * (h + prev)
    f[20:30] = h.mean(axis=0)
    f[30:40] = h.max(axis=0)
    return f.astype(np.float32)


def config_features_ref(coords: np.ndarray) -> np.ndarray:
    """fp32 restatement of rapp_mlp.cu:config_features (for the reference forward)."""
    c = np.asarray(coords, dtype=np.float64)
    f32 = np.float32
    b = np.clip(c[:, 0].astype(f32), f32(1), f32(512))
    s = np.clip(c[:, 1].astype(f32), f32(1), f32(100))
    q = np.clip(c[:, 2].astype(f32), f32(1), f32(100))
    cols = [b * f32(1 / 32), s * f32(0.01), q * f32(0.01), f32(1) / b, f32(1) / s,
            f32(1) / q, np.log2(b) * f32(0.2), np.log2(s) * f32(0.15),
            np.log2(q) * f32(0.15), s * q * f32(1e-4), f32(1) / (s * q),
            b / s * f32(1 / 32), b / q * f32(1 / 32), b / (s * q), np.sqrt(b) * f32(0.2),
            np.ones_like(b)]
    return np.stack(cols, axis=1).astype(np.float32)


@dataclass
class MlpWeights:
    w1: np.ndarray  # [128][64]
    b1: np.ndarray
    w2: np.ndarray  # [128][128]
    b2: np.ndarray
    w3: np.ndarray  # [128]
    b3: float

    @staticmethod
    def random(seed: int = 0) -> "MlpWeights":
        rng = np.random.default_rng(seed)
        f = np.float32
        return MlpWeights(
            w1=(rng.standard_normal((HIDDEN, K0)) * math.sqrt(2.0 / K0)).astype(f),
            b1=(rng.standard_normal(HIDDEN) * 0.05).astype(f),
            w2=(rng.standard_normal((HIDDEN, HIDDEN)) * math.sqrt(2.0 / HIDDEN)).astype(f),
            b2=(rng.standard_normal(HIDDEN) * 0.05).astype(f),
            w3=(rng.standard_normal(HIDDEN) * math.sqrt(1.0 / HIDDEN) * 0.5).astype(f),
            b3=float(math.log(20.0)))


class LearnedPerfModel:
    """PerfModel (hs/perf.py:23-31) backed by the fused tcgen05 MLP: one instance serves
    several models (graph features uploaded once); `for_model(name)` gives the per-function
    view with predict_latency / throughput."""

    def __init__(self, models: dict, weights: Optional[MlpWeights] = None, *,
                 device: int | None = None):
        self.names = list(models)
        self.weights = weights or MlpWeights.random(0)
        self.graph = np.stack([graph_features(ops) for ops in models.values()]).astype(np.float32)
        self.ctx = _lib.Context.get(device)
        w = self.weights
        h = _lib.c_vp()
        arrs = [np.ascontiguousarray(a, dtype=np.float32)
                for a in (self.graph, w.w1, w.b1, w.w2, w.b2, w.w3)]
        self._keep = arrs
        _lib.check(_lib.load().rapp_mlp_create(
            self.ctx.handle, len(self.names), *[a.ctypes.data for a in arrs],
            ctypes.c_float(w.b3), ctypes.byref(h)), "LearnedPerfModel")
        self._h = h

    @classmethod
    def zoo(cls, seed: int = 0, device: int | None = None) -> "LearnedPerfModel":
        return cls({k: f() for k, f in ZOO.items()}, MlpWeights.random(seed), device=device)

    def close(self) -> None:
        """Frees the device model now (also done when it is garbage-collected)."""
        h = getattr(self, "_h", None)
        self._h = None
        lib = getattr(_lib, "_lib", None) if _lib is not None else None
        if h is not None and lib is not None:
            lib.rapp_mlp_destroy(h)

    def __del__(self):
        self.close()

    def predict_many_dev(self, model: int, coords, out, *, stream=None):
        """Device API: coords (n, 3) float64 CUDA tensor -> out (n) float64 latency ms."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(coords.device).cuda_stream
        _lib.check(_lib.load().rapp_mlp_predict_dev(self._h, int(model), coords.data_ptr(),
                                                    int(coords.shape[0]), out.data_ptr(),
                                                    stream), "predict")
        return out

    def predict_many(self, model: int, coords: np.ndarray, out=None) -> np.ndarray:
        """Host API: (n, 3) float64 -> (n) latency ms through the chunked, stream-overlapped
        copy-in / kernel / copy-out pipeline (page-locked buffers are DMA'd directly)."""
        c = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 3)
        if out is None:
            out = np.empty(c.shape[0], dtype=np.float64)
        _lib.check(_lib.load().rapp_mlp_predict_host(self._h, int(model), _lib.dptr(c),
                                                     c.shape[0], _lib.dptr(out)), "predict")
        return out

    def search_dev(self, model_of_fn, targets, batches, sms, quota_step: int = 10, *,
                   stream=None):
        """most_efficient_config over the learned predictions for many functions at once
        (hs/perf.py:104-145 semantics on this model's rps): CUDA tensors model_of_fn (int32),
        targets (float64), batches / sms (float64, sorted) -> packed keys (uint64 as int64)."""
        import torch
        dev = targets.device
        n = int(targets.shape[0])
        if not 1 <= quota_step <= 100:
            raise ValueError("quota_step must be in [1, 100]")
        keys = torch.empty(n, dtype=torch.int64, device=dev)
        scratch = torch.empty(2 * n, dtype=torch.int64, device=dev)
        if stream is None:
            stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.load().rapp_mlp_search_dev(
            self._h, n, model_of_fn.data_ptr(), targets.data_ptr(), int(batches.shape[0]),
            batches.data_ptr(), int(sms.shape[0]), sms.data_ptr(), int(quota_step),
            keys.data_ptr(), scratch.data_ptr(), stream), "search")
        return keys

    def search(self, model_of_fn, targets, batches=(1, 2, 4, 8, 16, 32),
               sms=tuple(range(1, 101)), quota_step: int = 10) -> list[tuple[int, int, int]]:
        """Host API: one (b, s, q) per function."""
        import torch
        t = np.ascontiguousarray(targets, dtype=np.float64)
        if np.any(t <= 0):
            raise ValueError("target_rps must be positive")
        idx = [self.names.index(m) if isinstance(m, str) else int(m) for m in model_of_fn]
        dev = torch.device("cuda", self.ctx.device)
        bl = sorted({int(b) for b in batches})
        sl = sorted({int(s) for s in sms})
        keys = self.search_dev(torch.tensor(idx, dtype=torch.int32, device=dev),
                               torch.from_numpy(t).to(dev),
                               torch.tensor(bl, dtype=torch.float64, device=dev),
                               torch.tensor(sl, dtype=torch.float64, device=dev), quota_step)
        out = []
        for k in keys.cpu().numpy().view(np.uint64).tolist():
            out.append((bl[k & 0xFFF], sl[(k >> 20) & 0xFFF], (k >> 12) & 0xFF))
        return out

    def for_model(self, name: str) -> "_ModelView":
        return _ModelView(self, self.names.index(name))

    # -- the fp32 reference forward (test infrastructure for the parity-unpinned path) --
    def effective_weights(self):
        """The weights the kernel multiplies (rapp_mlp_create): biases on the constant
        feature (55) / constant hidden unit (127), the constant units fed 1.0."""
        w = self.weights
        c_in, c_h = N_GRAPH + N_CFG - 1, HIDDEN - 1
        e1 = w.w1.astype(np.float32).copy()
        e1[:, c_in] = w.b1
        e1[c_h, :] = 0.0
        e1[c_h, c_in] = 1.0
        e2 = w.w2.astype(np.float32).copy()
        e2[:, c_h] = w.b2
        e2[c_h, :] = 0.0
        e2[c_h, c_h] = 1.0
        e3 = w.w3.astype(np.float32).copy()
        e3[c_h] = w.b3
        return e1, e2, e3

    def reference_forward(self, model: int, coords: np.ndarray) -> np.ndarray:
        """fp32 forward of the same BF16 operands (x, weights and h1 rounded to BF16; h2 stays
        fp32: the output layer runs on the CUDA cores, rapp_mlp.cu RAPP_MLP_L3_FP32)."""
        import torch
        bf = torch.bfloat16
        e1, e2, e3 = (torch.from_numpy(a).to(bf).float() for a in self.effective_weights())
        x = np.zeros((len(coords), K0), dtype=np.float32)
        x[:, :N_GRAPH] = self.graph[model]
        x[:, N_GRAPH:N_GRAPH + N_CFG] = config_features_ref(coords)
        X = torch.from_numpy(x).to(bf).float()
        h1 = torch.relu(X @ e1.T).to(bf).float()
        h2 = torch.relu(h1 @ e2.T)
        y = h2 @ e3
        return torch.exp(torch.clamp(y, max=80.0)).double().numpy()


class _ModelView:
    """PerfModel protocol for one model of a LearnedPerfModel."""

    def __init__(self, lm: LearnedPerfModel, index: int):
        self.lm, self.index = lm, index
        self.function_id = lm.names[index]

    def predict_latency(self, batch: float, sm_percent: float, quota_percent: float) -> float:
        c = np.array([[float(batch), float(sm_percent), float(quota_percent)]])
        return float(self.lm.predict_many(self.index, c)[0])

    def throughput(self, batch: float, sm_percent: float, quota_percent: float) -> float:
        return batch / (self.predict_latency(batch, sm_percent, quota_percent) / 1000.0)

    def most_efficient_config(self, target_rps: float, *, quota_step: int = 10,
                              batches=None, sms=tuple(range(1, 101))):
        """hs/perf.py:104-145 over this model's predictions (lattice batches x sms x quota
        steps; batches default to 1..32 powers of two)."""
        if target_rps <= 0:
            raise ValueError("target_rps must be positive")
        return self.lm.search([self.index], [target_rps],
                              batches=batches or (1, 2, 4, 8, 16, 32), sms=sms,
                              quota_step=quota_step)[0]
