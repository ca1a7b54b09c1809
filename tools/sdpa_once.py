"""One cuDNN SDPA causal fwd+bwd (for ncu inspection of the library kernels)."""
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

n, h, d = 32768, 32, 128
q, k, v, do = ((torch.rand(1, h, n, d, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(4))
with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
    qq, kk, vv = (t.clone().requires_grad_() for t in (q, k, v))
    for _ in range(2):
        o = F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
        o.backward(do)
torch.cuda.synchronize()
print("ok")
