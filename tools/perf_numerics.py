"""Throughput of the float64 numerics kernels (csrc/bb_numerics.cu) on one GPU: the fp64 GEMM
(TFLOP/s) and the HBM-bound row kernels (GB/s of algorithmic traffic), CUDA-event timed."""
import json

import torch

from paper_2509_19836_b200 import numerics as F


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3


dev = torch.device("cuda:0")
n = 4096
a, b = (torch.rand(n, n, dtype=torch.float64, device=dev) for _ in range(2))
t = timed(lambda: F.matmul(a, b))
rows, cols = 16384, 16384
s = torch.randn(rows, cols, dtype=torch.float64, device=dev)
lse = F.row_logsumexp(s)
t_lse = timed(lambda: F.row_logsumexp(s))
t_exp = timed(lambda: F.exp_shifted(s, lse))
print(json.dumps({"matmul_f64_4096_tflops": 2 * n**3 / t / 1e12,
                  "row_logsumexp_gbs": rows * cols * 8 / t_lse / 1e9,
                  "exp_shifted_gbs": 2 * rows * cols * 8 / t_exp / 1e9}))
