"""Host <-> device movement for the NumPy drop-in API (make_device_states, shard_rows,
backward_grads, forward_results): burstsim callers hand in and get back NumPy arrays
(float64 results), so every call crosses PCIe.  Pageable copies plus a single-threaded host
cast ran at ~2-5 GB/s (backward_grads of one 128K x 32 x 128 tensor: 1.2 s); here the bytes go
through two reusable pinned staging buffers on a copy stream -- the copy engine moves chunk
c+1 while the host casts chunk c with torch's thread pool -- ~10x faster (tools/d2h_f64.py).

Values are unchanged: the host casts are exact (fp32 -> fp64) or the same float32 rounding
NumPy's astype performs (fp64 -> fp32, round to nearest even)."""

from __future__ import annotations

import numpy as np
import torch

_STAGE_BYTES = 128 << 20
_stages: dict = {}  # device index -> (two pinned uint8 buffers, copy stream, two events)


def _stage(dev: torch.device):
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    s = _stages.get(key)
    if s is None:
        bufs = [torch.empty(_STAGE_BYTES, dtype=torch.uint8).pin_memory() for _ in range(2)]
        s = (bufs, torch.cuda.Stream(dev), [torch.cuda.Event(), torch.cuda.Event()])
        _stages[key] = s
    return s


def empty_f64(t: torch.Tensor) -> np.ndarray:
    """A float64 NumPy array shaped like ``t`` whose pages are already resident: written once
    (zeros, torch's thread pool) so the copy into it later does not stop on first-touch page
    faults.  Called while the GPU still runs the kernels that produce ``t``, this host work
    overlaps them (``backward_grads``)."""
    out = np.empty(tuple(t.shape), dtype=np.float64)
    torch.from_numpy(out).zero_()
    return out


def to_host_f64(t: torch.Tensor, out: np.ndarray | None = None) -> np.ndarray:
    """float64 NumPy copy of a CUDA float tensor (any float dtype, made contiguous first),
    into ``out`` if given (a C-contiguous float64 array of ``t``'s shape)."""
    if out is not None and (out.shape != tuple(t.shape) or out.dtype != np.float64 or not out.flags.c_contiguous):
        raise ValueError(f"out must be a C-contiguous float64 array of shape {tuple(t.shape)}")
    if not t.is_cuda:
        a = t.detach().double().numpy()
        if out is None:
            return a
        out[...] = a
        return out
    src = t.detach()
    if src.dtype != torch.float32:
        src = src.float()
    src = src.contiguous().reshape(-1)
    if out is None:
        out = np.empty(tuple(t.shape), dtype=np.float64)
    dst = torch.from_numpy(out).reshape(-1)
    n = src.numel()
    if n == 0:
        return out
    bufs, stream, events = _stage(t.device)
    per = _STAGE_BYTES // 4
    chunks = [(i, min(n, i + per)) for i in range(0, n, per)]
    stream.wait_stream(torch.cuda.current_stream(t.device))

    def issue(c):
        lo, hi = chunks[c]
        with torch.cuda.stream(stream):
            bufs[c % 2].view(torch.float32)[: hi - lo].copy_(src[lo:hi], non_blocking=True)
            events[c % 2].record(stream)

    issue(0)
    for c, (lo, hi) in enumerate(chunks):
        if c + 1 < len(chunks):
            issue(c + 1)  # its buffer was read by chunk c - 1's host cast, which has returned
        events[c % 2].synchronize()
        dst[lo:hi].copy_(bufs[c % 2].view(torch.float32)[: hi - lo])
    return out


def to_device(x: np.ndarray, dev: torch.device, dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """CUDA copy of a NumPy array as ``dtype`` (float32 or bfloat16): the host casts each chunk
    into pinned staging, the copy engine uploads it while the next chunk is cast."""
    a = np.ascontiguousarray(x)
    src = torch.from_numpy(a).reshape(-1)
    out = torch.empty(a.shape, dtype=dtype, device=dev)
    dst = out.reshape(-1)
    n = src.numel()
    if n == 0:
        return out
    bufs, stream, events = _stage(dev)
    for e in events:  # an earlier upload may still be reading the staging buffers
        e.synchronize()
    esize = torch.empty((), dtype=dtype).element_size()
    per = _STAGE_BYTES // esize
    compute = torch.cuda.current_stream(dev)
    stream.wait_stream(compute)  # ``out`` is allocated on the compute stream
    for c, lo in enumerate(range(0, n, per)):
        hi = min(n, lo + per)
        b = c % 2
        if c >= 2:
            events[b].synchronize()  # the upload that last read this staging buffer has finished
        bufs[b].view(dtype)[: hi - lo].copy_(src[lo:hi])  # host cast (torch thread pool)
        with torch.cuda.stream(stream):
            dst[lo:hi].copy_(bufs[b].view(dtype)[: hi - lo], non_blocking=True)
            events[b].record(stream)
    compute.wait_stream(stream)
    out.record_stream(stream)
    return out
