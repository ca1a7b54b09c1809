"""Rate of single ring-step kernels for given (query device, key device) pairs of a layout, on
one GPU (the shards are synthetic; only the mask geometry matters).  Developer tool.

    python tools/pair_rate.py --seq 1048576 --devices 2 --heads 8 --pairs 1,1 2,1
"""
import argparse
import math
import os
import sys

import torch

from paper_2509_19836_b200 import kernels as K
from paper_2509_19836_b200.masks import causal_mask
from paper_2509_19836_b200.partitioning import ShardLayout, pair_count_matrix

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=1 << 20)
ap.add_argument("--devices", type=int, default=2)
ap.add_argument("--heads", type=int, default=8)
ap.add_argument("--layout", default="zigzag")
ap.add_argument("--pairs", nargs="+", default=["1,1", "2,1"])
args = ap.parse_args()
dev = torch.device("cuda")
layout = ShardLayout(args.layout, args.seq, args.devices)
mask = causal_mask()
dm = K.device_mask(mask, dev)
counts = pair_count_matrix(layout, mask)
n, h, d = layout.shard_size, args.heads, 128
q, k, v, do = ((torch.rand(n, h, d, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(4))
o = torch.zeros(n, h, d, device=dev)
lse = torch.zeros(h, n, device=dev)
delta = torch.zeros(h, n, device=dev)
dq, dk, dv = (torch.zeros(n, h, d, device=dev) for _ in range(3))
for pr in args.pairs:
    i, j = (int(x) for x in pr.split(","))
    pairs = counts[i - 1, j - 1] * h
    for name, fn, f in (("fwd", lambda: K.attn_fwd_step(q, k, v, o, lse, layout, dm, i, j, 1 / math.sqrt(d)), 4),
                        ("bwd", lambda: K.attn_bwd_step(q, k, v, do, lse, delta, dq, dk, dv, layout, dm, i, j,
                                                        1 / math.sqrt(d)), 10)):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(0) as clk:
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
        t = a.elapsed_time(b) / 1e3
        print(f"pair q{i} x k{j} {name}: {t * 1e3:.1f} ms  {f * d * pairs / t / 1e12:.0f} TFLOP/s  clocks {clk.summary()}",
              flush=True)
