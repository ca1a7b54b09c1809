"""One cfg5 fused LM head pass (131072 tokens, V=131072, D=4096, B_s=8192) for an ncu launch
list: which of the five kernels per row tile take the time.  Developer tool."""
import math

import torch

from paper_2509_19836_b200.lmhead import FusionConfig, fused_lmhead_loss

n, v, d = 131072, 131072, 4096
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(77)
h = (torch.rand(n, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
w = ((torch.rand(v, d, device=dev, generator=g) * 2 - 1) / math.sqrt(d)).to(torch.bfloat16)
y = torch.randint(0, v, (n,), device=dev, generator=g)
cfg = FusionConfig(8192, 4096)
for _ in range(2):
    fused_lmhead_loss(h, w, y, cfg)
torch.cuda.synchronize()
