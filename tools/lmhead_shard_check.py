"""torchrun check of the sequence-sharded LM head on N GPUs (tests/test_lmhead_sharded.py):
each rank holds a token shard, dW and the loss are all-reduced over NCCL; rank 0 compares with
the fp64 oracle on the whole sequence."""
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import burst_oracle as O  # noqa: E402
from paper_2509_19836_b200 import lmhead as L  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
n, v, d = 1536, 4099, 256
rng = np.random.default_rng(11)
h = torch.from_numpy(rng.uniform(-1, 1, (n, d))).float().to(torch.bfloat16)
w = torch.from_numpy(rng.uniform(-1, 1, (v, d)) / math.sqrt(d)).float().to(torch.bfloat16)
y = rng.integers(0, v, n)
rows = np.array_split(np.arange(n), world)[rank]
res = L.sharded_fused_lmhead_loss(h[rows].to(dev), w.to(dev), torch.from_numpy(y[rows]).to(dev), L.FusionConfig(256, 1024))
loss, dh, dw = O.naive_lmhead(h.double().numpy(), w.double().numpy(), y)
ok = abs(res.total_loss - loss.sum()) < 2e-3 * n
ok &= float(np.abs(res.loss.double().cpu().numpy() - loss[rows]).max()) < 2e-3
ok &= float(np.linalg.norm(res.dh.double().cpu().numpy() - dh[rows]) / np.linalg.norm(dh[rows])) < 1e-2
ok &= float(np.linalg.norm(res.dw.double().cpu().numpy() - dw) / np.linalg.norm(dw)) < 1e-2
flag = torch.tensor([1 if ok else 0], device=dev)
dist.all_reduce(flag, op=dist.ReduceOp.MIN)
if rank == 0:
    print("lmhead shard check ok" if int(flag.item()) == 1 else "lmhead shard check FAIL", flush=True)
dist.destroy_process_group()
sys.exit(0 if int(flag.item()) == 1 else 1)
