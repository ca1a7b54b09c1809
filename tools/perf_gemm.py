"""Time the tcgen05 GEMM (LM-head building block) for each operand-major combination."""

import sys

import torch

from paper_2509_19836_b200 import kernels as K

dev = torch.device("cuda:0")
m = n = k = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.randn(m, k, device=dev).to(torch.bfloat16)
b = torch.randn(n, k, device=dev).to(torch.bfloat16)
c = torch.empty(m, n, device=dev)
for a_mn in (False, True):
    for b_mn in (False, True):
        A = a.t().contiguous() if a_mn else a
        B = b.t().contiguous() if b_mn else b
        K.gemm(A, B, c, m, n, k, a_mn, b_mn, False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            K.gemm(A, B, c, m, n, k, a_mn, b_mn, False)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 5 / 1e3
        print(f"gemm {m}x{n}x{k} a_mn={a_mn} b_mn={b_mn}: {t*1e3:.3f} ms {2*m*n*k/t/1e12:.1f} TFLOP/s", flush=True)
ref = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
e0.record()
for _ in range(5):
    torch.matmul(a, b.t(), out=ref)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 5 / 1e3
print(f"cublas bf16 {m}x{n}x{k}: {2*m*n*k/t/1e12:.1f} TFLOP/s")
