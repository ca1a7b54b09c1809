"""Forward probe with a single live query tile per CTA (n_q = 128): the softmax timeline of
one warpgroup without its ping-pong partner (BB_PROBE=1)."""
import math
import os
import sys

os.environ["BB_PROBE"] = "1"
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_19836_b200 import _native as N  # noqa: E402
from paper_2509_19836_b200 import kernels as K  # noqa: E402
from paper_2509_19836_b200.masks import full_mask  # noqa: E402
from paper_2509_19836_b200.partitioning import ShardLayout  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 128
nk, h, d = 32768, 8, 128
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
q = (torch.rand(nq, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
k = (torch.rand(nk, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
v = (torch.rand(nk, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
o = torch.zeros(nq, h, d, device=dev)
lse = torch.full((h, nq), float("-inf"), device=dev)
layout = ShardLayout("contiguous", nk, 1)
# a contiguous layout with n_q != n_k: q rows are token ids 1..nq, all keys visible (full mask)
K.attn_fwd_step(q, k, v, o, lse, layout, K.device_mask(full_mask(), dev), 1, 1, 1 / math.sqrt(d))
torch.cuda.synchronize()
buf = np.zeros(4096, dtype=np.int64)
N.check(N.load().bb_debug_probe(buf.ctypes.data, 4096))
t = buf[512:1024].reshape(16, 32)
base = t[t > 0].min()
names = {4: "m:K?", 5: "m:K", 7: "m:P0", 9: "m:P1", 16: "s0:S?", 17: "s0:S", 22: "s0:ldS?", 23: "s0:ldS", 18: "s0:pv", 20: "s0:Pstored", 21: "s0:fenced", 19: "s0:P",
         24: "s1:S?", 25: "s1:S", 30: "s1:ldS?", 31: "s1:ldS", 26: "s1:pv", 28: "s1:Pstored", 29: "s1:fenced", 27: "s1:P"}
for it in range(16):
    print(it, " ".join(f"{names[s]}={t[it, s]-base}" for s in sorted(names) if t[it, s] > 0))
