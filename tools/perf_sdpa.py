"""Library comparison point (not the product): torch SDPA (cuDNN / flash backends) fwd and
fwd+bwd on the cfg2 shape, CUDA-event timed, TFLOP/s with the same causal FLOP count as
tools/perf_attn.py.   python tools/perf_sdpa.py [--n 131072] [--heads 32]"""
import argparse

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=131072)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--iters", type=int, default=3)
args = ap.parse_args()
n, h, d = args.n, args.heads, args.d
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = ((torch.rand(1, h, n, d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(4))
pairs = n * (n + 1) // 2
for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION)):
    try:
        with sdpa_kernel([be]):
            qq, kk, vv = (t.clone().requires_grad_() for t in (q, k, v))
            for _ in range(2):
                o = F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
                o.backward(do)
            torch.cuda.synchronize()
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            tf = tb = 0.0
            for _ in range(args.iters):
                a.record()
                o = F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
                b.record()
                o.backward(do)
                c.record()
                torch.cuda.synchronize()
                tf += a.elapsed_time(b)
                tb += b.elapsed_time(c)
            tf /= args.iters
            tb /= args.iters
            print(f"sdpa[{name}] fwd {tf:.2f} ms {4 * d * h * pairs / tf / 1e9:.1f} TF/s   bwd {tb:.2f} ms {10 * d * h * pairs / tb / 1e9:.1f} TF/s")
    except Exception as e:  # noqa: BLE001
        print(f"sdpa[{name}] unavailable: {type(e).__name__}: {str(e)[:120]}")
