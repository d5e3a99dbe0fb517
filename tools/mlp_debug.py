"""Compares the MLP kernel's first-tile accumulators with X.W1^T / H.W2^T (diagnostics)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_01968_b200 import _lib, learned  # noqa: E402

lm = learned.LearnedPerfModel.zoo(seed=3)
rng = np.random.default_rng(0)
n = 128
c = np.column_stack([rng.uniform(1, 32, n), rng.uniform(1, 100, n), rng.uniform(1, 100, n)])
dc = torch.from_numpy(c).cuda()
out = torch.empty(n, dtype=torch.float64, device="cuda")
acc = torch.zeros(2 * 128 * 128, dtype=torch.float32, device="cuda")
_lib.check(_lib.load().rapp_mlp_debug_dev(lm._h, 0, dc.data_ptr(), n, out.data_ptr(),
                                          acc.data_ptr(), torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
a = acc.cpu().numpy().reshape(2, 128, 128)
bf = torch.bfloat16
w = lm.weights
x = np.zeros((n, 64), dtype=np.float32)
x[:, :40] = lm.graph[0]
x[:, 40:56] = learned.config_features_ref(c)
X = torch.from_numpy(x).to(bf).float()
e1, e2, e3 = (torch.from_numpy(a).to(bf).float() for a in lm.effective_weights())
ref1 = (X @ e1.T).numpy()
print("acc1 vs ref1: max abs diff", np.abs(a[0] - ref1).max(), "ref scale", np.abs(ref1).max())
print("acc1[0,:8]", a[0, 0, :8])
print("ref1[0,:8]", ref1[0, :8])
print("acc1[9,:8]", a[0, 9, :8])
print("ref1[9,:8]", ref1[9, :8])
# does acc1 match a row/col permutation?
for name, cand in (("transpose", ref1.T),):
    print(name, np.abs(a[0] - cand).max())
h1 = torch.relu(torch.from_numpy(ref1)).to(bf).float()
ref2 = (h1 @ e2.T).numpy()
print("acc2 vs ref2: max abs diff", np.abs(a[1] - ref2).max(), "ref scale", np.abs(ref2).max())
print("out[:8]", out[:8].cpu().numpy())
print("ref[:8]", lm.reference_forward(0, c)[:8])
