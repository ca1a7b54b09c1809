"""cfg5 measurement: fused LM head + cross entropy on one B200 (one sequence shard of the 1M-token
job over 8 GPUs: 131072 tokens, V = 131072, D = 4096), 6*N*V*D FLOPs per step, plus the
sequence-selective checkpoint recompute of the attention layer (s = 0.5) when --ckpt is given.

    python tools/bench_lmhead.py [--tokens 131072] [--vocab 131072] [--dim 4096] [--rows 8192]
"""

import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_19836_b200 import _native  # noqa: E402
from paper_2509_19836_b200 import kernels as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=131072)
ap.add_argument("--vocab", type=int, default=131072)
ap.add_argument("--dim", type=int, default=4096)
ap.add_argument("--rows", type=int, default=8192, help="B_s row tile")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=1)
args = ap.parse_args()

dev = torch.device("cuda:0")
_native.load()
n, v, d = args.tokens, args.vocab, args.dim
g = torch.Generator(device=dev).manual_seed(0)
h = (torch.rand(n, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
w = ((torch.rand(v, d, device=dev, generator=g) * 2 - 1) / math.sqrt(d)).to(torch.bfloat16)
y = torch.randint(0, v, (n,), device=dev, generator=g)
loss = torch.empty(n, device=dev)
dh = torch.empty(n, d, device=dev)
dw = torch.zeros(v, d, device=dev)
ws = torch.empty(K.lmhead_workspace_bytes(n, v, d, args.rows), dtype=torch.uint8, device=dev)


def step():
    dw.zero_()
    K.lmhead_fused(h, w, y, loss, dh, dw, args.rows, 4096, ws)


for _ in range(args.warmup):
    step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(args.steps):
    step()
b.record()
torch.cuda.synchronize()
t = a.elapsed_time(b) / 1e3 / args.steps
flops = 6.0 * n * v * d
print(json.dumps({
    "workload": f"cfg5 fused LM head + CE: {n} tokens (one of 8 sequence shards of 2^20), V={v}, D={d}, B_s={args.rows}",
    "tflops": flops / t / 1e12, "ms_per_step": t * 1e3, "flops_per_step": flops,
    "loss_mean": float(loss.mean()), "logits_scratch_bytes": int(ws.numel()),
}))
