"""Quick kernel timing: one fwd step and one bwd step of cfg2 (N=128K causal, 32 heads,
d=128, G=1) with CUDA events.  Developer tool; bench.py is the contract."""

import argparse
import math
import time

import torch

from paper_2509_19836_b200 import kernels as K
from paper_2509_19836_b200.masks import causal_mask, full_mask
from paper_2509_19836_b200.partitioning import ShardLayout

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=131072)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--mask", default="causal")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--halves", action="store_true", help="also time the bwd step split by kv heads (A, B, B, A)")
args = ap.parse_args()

dev = torch.device("cuda:0")
n, h, d = args.n, args.heads, args.d
mask = causal_mask() if args.mask == "causal" else full_mask()
layout = ShardLayout("contiguous", n, 1)
g = torch.Generator(device=dev).manual_seed(0)
q = (torch.rand(n, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
k = (torch.rand(n, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
v = (torch.rand(n, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
do = (torch.rand(n, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
o = torch.zeros(n, h, d, device=dev)
lse = torch.full((h, n), float("-inf"), device=dev)
delta = torch.empty(h, n, device=dev)
dq = torch.zeros(n, h, d, device=dev)
dk = torch.zeros(n, h, d, device=dev)
dv = torch.zeros(n, h, d, device=dev)
dm = K.device_mask(mask, dev)
scale = 1 / math.sqrt(d)
pairs = n * (n + 1) // 2 if args.mask == "causal" else n * n


def fwd():
    o.zero_()
    lse.fill_(float("-inf"))
    K.attn_fwd_step(q, k, v, o, lse, layout, dm, 1, 1, scale)


def bwd():
    K.bwd_preprocess(do, o, delta)
    K.attn_bwd_step(q, k, v, do, lse, delta, dq, dk, dv, layout, dm, 1, 1, scale)


for name, fn, flops in (("fwd", fwd, 4 * d * h * pairs), ("bwd", bwd, 10 * d * h * pairs)):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    t = min(ts)
    print(f"{name}: {t*1e3:.2f} ms  {flops/t/1e12:.1f} TFLOP/s  (n={n} h={h} d={d} {args.mask})", flush=True)

if args.halves:  # the ring's own-step split: is half B as fast as half A on its own?
    K.bwd_preprocess(do, o, delta)
    for heads in ((0, h // 2), (h // 2, h), (h // 2, h), (0, h // 2)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        K.attn_bwd_step(q, k, v, do, lse, delta, dq, dk, dv, layout, dm, 1, 1, scale, kv_heads=heads)
        b.record()
        torch.cuda.synchronize()
        print(f"bwd kv heads {heads}: {a.elapsed_time(b):.2f} ms", flush=True)
