"""Does cudaMemsetAsync (and torch's zero_) overlap a compute-bound kernel, i.e. run off the
SMs?  Times the forward kernel (64K causal, 32 heads) alone, a 4 GB zero alone, and both on
two streams.  Developer tool."""

import ctypes as C
import glob
import math
import os

import torch

from paper_2509_19836_b200 import kernels as K
from paper_2509_19836_b200.masks import causal_mask
from paper_2509_19836_b200.partitioning import ShardLayout

lib = None
for pat in ("/usr/local/cuda/lib64/libcudart.so*",
            os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*")):
    for f in sorted(glob.glob(pat)):
        try:
            lib = C.CDLL(f)
            break
        except OSError:
            pass
    if lib:
        break

dev = torch.device("cuda:0")
n, h, d = 65536, 32, 128
layout = ShardLayout("contiguous", n, 1)
q, k, v = ((torch.rand(n, h, d, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(3))
o = torch.zeros(n, h, d, device=dev)
lse = torch.full((h, n), float("-inf"), device=dev)
dm = K.device_mask(causal_mask(), dev)
buf = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def fwd():
    K.attn_fwd_step(q, k, v, o, lse, layout, dm, 1, 1, 1 / math.sqrt(d))


def memset():
    rc = lib.cudaMemsetAsync(C.c_void_p(buf.data_ptr()), 0, C.c_size_t(buf.numel()), C.c_void_p(s2.cuda_stream))
    assert rc == 0, rc


def zero_():
    buf.zero_()


zeros = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)


def d2d_copy():  # same-device copies from a zero buffer: copy engine or SMs?
    for off in range(0, buf.numel(), zeros.numel()):
        rc = lib.cudaMemcpyAsync(C.c_void_p(buf.data_ptr() + off), C.c_void_p(zeros.data_ptr()),
                                 C.c_size_t(zeros.numel()), 3, C.c_void_p(s2.cuda_stream))
        assert rc == 0, rc


def timed(stream, fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record(stream)
        fn()
        b.record(stream)
    return a, b


for name, z in (("cudaMemsetAsync", memset), ("torch zero_", zero_), ("D2D cudaMemcpyAsync", d2d_copy)):
    for _ in range(2):
        torch.cuda.synchronize()
        fa, fb = timed(s1, fwd)
        torch.cuda.synchronize()
        za, zb = timed(s2, z)
        torch.cuda.synchronize()
        alone = (fa.elapsed_time(fb), za.elapsed_time(zb))
        fa, fb = timed(s1, fwd)
        za, zb = timed(s2, z)
        torch.cuda.synchronize()
        both = (fa.elapsed_time(fb), za.elapsed_time(zb))
    print(f"{name}: alone fwd {alone[0]:.2f} ms, 4 GB zero {alone[1]:.3f} ms; together fwd {both[0]:.2f} ms, zero {both[1]:.3f} ms",
          flush=True)
