"""How fast can a [131072, 32, 128] fp32 device tensor become a float64 NumPy array (the
drop-in API's backward_grads)?  Variants: host cast (the current path), device cast + copy into
a fresh array, the same with MADV_HUGEPAGE on the destination.  Developer tool."""

import ctypes
import mmap
import time

import numpy as np
import torch

print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(), flush=True)
libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
MADV_HUGEPAGE = 14

t = torch.rand(131072, 32, 128, device="cuda")


def timed(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a = fn()
    torch.cuda.synchronize()
    print(f"{name}: {time.perf_counter() - t0:.3f} s", flush=True)
    return a


def host_cast():
    return t.float().cpu().double().numpy()


def dev_cast():
    a = np.empty(t.shape, dtype=np.float64)
    torch.from_numpy(a).copy_(t.double())
    return a


def dev_cast_huge():
    nbytes = t.numel() * 8
    buf = mmap.mmap(-1, nbytes + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    addr = ctypes.addressof(ctypes.c_char.from_buffer(buf))
    libc.madvise(ctypes.c_void_p(addr), nbytes, MADV_HUGEPAGE)
    a = np.frombuffer(buf, dtype=np.float64, count=t.numel()).reshape(t.shape)
    torch.from_numpy(a).copy_(t.double())
    return a


STAGE = 64 << 20  # floats per staging buffer (256 MB)
pinned = [torch.empty(STAGE, dtype=torch.float32).pin_memory() for _ in range(2)]
copy_stream = torch.cuda.Stream()


def staged():
    """fp32 chunks -> pinned staging (copy engine, async) -> multi-threaded host cast into the
    float64 destination; two staging buffers so the next chunk's D2H overlaps this chunk's cast."""
    a = np.empty(t.shape, dtype=np.float64)
    src, dst = t.reshape(-1), torch.from_numpy(a).reshape(-1)
    n = src.numel()
    events = [torch.cuda.Event(), torch.cuda.Event()]
    chunks = [(i, min(n, i + STAGE)) for i in range(0, n, STAGE)]
    copy_stream.wait_stream(torch.cuda.current_stream())

    def issue(c):
        lo, hi = chunks[c]
        with torch.cuda.stream(copy_stream):
            pinned[c % 2][: hi - lo].copy_(src[lo:hi], non_blocking=True)
            events[c % 2].record(copy_stream)

    issue(0)
    for c, (lo, hi) in enumerate(chunks):
        if c + 1 < len(chunks):
            if c >= 1:
                pass  # buffer (c+1)%2 was consumed by chunk c-1's cast, already finished (host order)
            issue(c + 1)
        events[c % 2].synchronize()
        dst[lo:hi].copy_(pinned[c % 2][: hi - lo])
    return a


print("threads", torch.get_num_threads(), flush=True)
for _ in range(2):
    ref = timed("host cast (current)", host_cast)
    e = timed("pinned staging + threaded host cast", staged)
    assert np.array_equal(ref, e)
    b = timed("device cast + copy", dev_cast)
    c = timed("device cast + copy, MADV_HUGEPAGE", dev_cast_huge)
    assert np.array_equal(ref, b) and np.array_equal(ref, c)
