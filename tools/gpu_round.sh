timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mlp -s 1 -c 1 -o gpurun_out/prof_mlp_r01e python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_2505_01968_b200 import learned
lm = learned.LearnedPerfModel.zoo()
n = 20_000_000
c = torch.rand((n,3), dtype=torch.float64, device='cuda') * torch.tensor([31.,99.,99.], dtype=torch.float64, device='cuda') + 1
o = torch.empty(n, dtype=torch.float64, device='cuda')
for _ in range(2): lm.predict_many_dev(0, c, o)
torch.cuda.synchronize()
" > /dev/null 2>&1
