"""Per-CTA timeline of one forward launch (probe build): prologue, main loop and epilogue
durations and the idle gap between consecutive CTAs on each SM.  Developer tool.

    python tools/variant.py probes BB_WITH_PROBES
    BB_LIB_PATH=tools/exp_lib/probes/libburst_b200.so python tools/cta_timeline.py --n 16384 --mask causal
"""
import argparse
import math
import os

os.environ["BB_PROBE"] = "1"
os.environ.setdefault("BB_LIB_PATH", "tools/exp_lib/probes/libburst_b200.so")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_19836_b200 import _native as N  # noqa: E402
from paper_2509_19836_b200 import kernels as K  # noqa: E402
from paper_2509_19836_b200.masks import causal_mask, full_mask  # noqa: E402
from paper_2509_19836_b200.partitioning import ShardLayout  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--mask", default="causal")
ap.add_argument("--kernel", default="fwd", choices=["fwd", "bwd"])
ap.add_argument("--merge", action="store_true", help="fwd: time a second step that merges into the first's (O, lse)")
args = ap.parse_args()
dev = torch.device("cuda")
n, h, d = args.n, args.heads, 128
layout = ShardLayout("contiguous", n, 1)
dm = K.device_mask(causal_mask() if args.mask == "causal" else full_mask(), dev)
q, k, v = ((torch.rand(n, h, d, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(3))
o = torch.zeros(n, h, d, device=dev)
lse = torch.full((h, n), float("-inf"), device=dev)
for _ in range(2):
    o.zero_()
    lse.fill_(float("-inf"))
    K.attn_fwd_step(q, k, v, o, lse, layout, dm, 1, 1, 1 / math.sqrt(d))
if args.merge and args.kernel == "fwd":
    K.attn_fwd_step(q, k, v, o, lse, layout, dm, 1, 1, 1 / math.sqrt(d))  # w_old != 0 everywhere
torch.cuda.synchronize()
if args.kernel == "bwd":
    do = (torch.rand(n, h, d, device=dev) * 2 - 1).to(torch.bfloat16)
    delta = torch.empty(h, n, device=dev)
    dq, dk, dv = (torch.zeros(n, h, d, device=dev) for _ in range(3))
    K.bwd_preprocess(do, o, delta)
    for _ in range(2):
        K.attn_bwd_step(q, k, v, do, lse, delta, dq, dk, dv, layout, dm, 1, 1, 1 / math.sqrt(d))
    torch.cuda.synchronize()
buf = np.zeros(65536, dtype=np.int64)
N.check(N.load().bb_debug_probe(buf.ctypes.data, 65536))
ctas = ((n + 255) // 256 if args.kernel == "fwd" else (n + 127) // 128) * h
ctas = min(ctas, (65536 - 4096) // 8)
rec = buf[4096: 4096 + ctas * 8].reshape(ctas, 8)
rec = rec[rec[:, 1] > 0]
base = rec[:, 1].min()
sm = rec[:, 0]
if args.kernel == "fwd":
    t0, t1, t2, t3, t4, t5, t6 = (rec[:, i] for i in range(1, 8))
    print(f"{len(rec)} CTAs on {len(set(sm.tolist()))} SMs, kernel span {(t3.max() - base) / 1e3:.1f} us")
    print(f"prologue  mean {np.mean(t1 - t0) / 1e3:.2f} us  max {np.max(t1 - t0) / 1e3:.2f}")
    print(f"main      mean {np.mean(t2 - t1) / 1e3:.2f} us")
    print(f"epilogue  mean {np.mean(t3 - t2) / 1e3:.2f} us  max {np.max(t3 - t2) / 1e3:.2f}")
    print(f"  query tile 1 loop ends after tile 0's by {np.mean(t4 - t2) / 1e3:.2f} us (mean)")
    end = t3
else:
    t0, t1, t2, t3, t4, t5 = (rec[:, i] for i in range(1, 7))
    print(f"{len(rec)} CTAs on {len(set(sm.tolist()))} SMs, kernel span {(t4.max() - base) / 1e3:.1f} us")
    print(f"prologue  mean {np.mean(t1 - t0) / 1e3:.2f} us  max {np.max(t1 - t0) / 1e3:.2f}")
    print(f"main      mean {np.mean(t2 - t1) / 1e3:.2f} us")
    print(f"dK/dV     mean {np.mean(t3 - t2) / 1e3:.2f} us (acc_full wait {np.mean(t5 - t2) / 1e3:.2f} us, "
          f"stores {np.mean(t3 - t5) / 1e3:.2f} us);  then exit {np.mean(t4 - t3) / 1e3:.2f} us")
    end = t4
gaps, busy, ends = [], [], []
for s_ in set(sm.tolist()):
    idx = np.argsort(t0[sm == s_])
    a, b = t0[sm == s_][idx], end[sm == s_][idx]
    gaps.extend((a[1:] - b[:-1]).tolist())
    busy.append(int(np.sum(b - a)))
    ends.append(int(b[-1] - base))
print(f"gap between CTAs on an SM: mean {np.mean(gaps) / 1e3:.2f} us  max {np.max(gaps) / 1e3:.2f}")
print(f"SM busy fraction: {np.sum(busy) / (len(busy) * (end.max() - base)):.3f}; last CTA end spread "
      f"{(max(ends) - min(ends)) / 1e3:.1f} us")
