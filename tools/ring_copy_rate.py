"""Why a ring push runs below the isolated probe: the same bidirectional copy-engine push of a
K/V payload (2 x 537 MB bf16 at 128K tokens / 2 ranks, 32 heads, d=128) into the ring's
Channel arena, issued (a) as raw copies of bench-like tensors, (b) through Channel.push with
its flags, (c) as raw copies of one fresh 1 GiB buffer (the probe's case).  Medians of 7.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563 tools/ring_copy_rate.py
"""

import ctypes as C
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_19836_b200 import _native as N  # noqa: E402
from paper_2509_19836_b200.peer import Channel  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    peer = 1 - rank
    n, h, d = 65536, 32, 128
    g = torch.Generator(device=dev).manual_seed(rank)
    k = (torch.rand(n, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    v = (torch.rand(n, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    flat = torch.empty(2 * k.numel() * 2, dtype=torch.uint8, device=dev)
    ch = Channel("kv", [(tuple(k.shape), k.dtype), (tuple(v.shape), v.dtype)], [None, peer], [None, peer], rank, world, dev)
    lib = N.load()
    s = torch.cuda.Stream(dev)
    nbytes = ch.payload_bytes
    out = {}

    def timed(fn):
        rates = []
        for _ in range(7):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / 1e3], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            rates.append(nbytes / float(t.item()) / 1e9)
        rates.sort()
        return {"median": rates[3], "best": rates[-1], "worst": rates[0]}

    def raw(srcs):
        def f():
            base = ch.peer_base[peer]
            for t, off in zip(srcs, ch.offsets):
                N.check(lib.bb_copy_async(C.c_void_p(base + off), C.c_void_p(t.data_ptr()), t.numel() * t.element_size(),
                                          C.c_void_p(s.cuda_stream)))
        return f

    def push():
        ch.begin()
        ch.push(1, [k, v], s)
        ch.release(1, s)  # I am also the receiver of the peer's push: hand my slot back

    out["raw_bench_tensors_GBps"] = timed(raw([k, v]))
    out["channel_push_GBps"] = timed(push)
    half = flat.numel() // 2
    out["raw_fresh_buffer_GBps"] = timed(raw([flat[:half], flat[half:]]))
    # (d) the same push right after ~1.5 s of dense bf16 GEMMs (the ring's pushes follow attention
    # kernels that hold the GPU at its power cap), and (e) pushes concurrent with those GEMMs
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)

    def heat(iters=600):
        for _ in range(iters):
            torch.mm(a, a)

    def push_after_heat():
        heat()
        torch.cuda.current_stream().synchronize()
        push()

    rates = []
    for _ in range(5):
        torch.cuda.synchronize()
        dist.barrier()
        heat()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.wait_stream(torch.cuda.current_stream())
        e0.record(s)
        push()
        e1.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 1e3], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rates.append(nbytes / float(t.item()) / 1e9)
    rates.sort()
    out["channel_push_after_gemms_GBps"] = {"median": rates[2], "best": rates[-1], "worst": rates[0]}
    rates = []
    for _ in range(5):
        torch.cuda.synchronize()
        dist.barrier()
        heat(200)  # GEMMs queued on the compute stream; the push runs beside them
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        push()
        e1.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 1e3], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rates.append(nbytes / float(t.item()) / 1e9)
    rates.sort()
    out["channel_push_beside_gemms_GBps"] = {"median": rates[2], "best": rates[-1], "worst": rates[0]}
    out["payload_bytes"] = nbytes
    if rank == 0:
        print(json.dumps(out), flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    ch.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
