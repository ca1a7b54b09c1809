"""Copy-engine rates between two ranks through the ring's own CUDA-IPC arenas (torchrun, 2 GPUs):
push (issued by the sender, writing the peer's arena) and pull (issued by the receiver, reading
the peer's arena), one and both directions, 1 and 2 streams, 1 GiB per copy.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 tools/p2p_ipc_bw.py
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
    n = 1 << 30
    peer = 1 - rank
    ch = Channel("bw", [((n,), torch.uint8)], [None, peer], [None, peer], rank, world, dev, slots=1)
    lib = N.load()
    local = torch.empty(n, dtype=torch.uint8, device=dev).fill_(rank + 1)
    streams = [torch.cuda.Stream(dev) for _ in range(2)]
    out = {}

    def run(kind, both, k, arena_dst=False, pieces=1):
        rates = []
        for _ in range(7):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cur = torch.cuda.current_stream()
            e0.record(cur)
            active = both or rank == 0
            if active:
                part = n // k
                mine = ch.base if arena_dst else local.data_ptr()  # pull target: my arena or a torch buffer
                for i in range(k):
                    s = streams[i]
                    s.wait_event(e0)
                    if kind == "push":  # my buffer -> the peer's arena
                        dst, src = ch.peer_base[peer] + i * part, local.data_ptr() + i * part
                    else:  # the peer's arena -> my buffer
                        dst, src = mine + i * part, ch.peer_base[peer] + i * part
                    piece = part // pieces  # several back-to-back copies on the stream (the ring's per-tensor copies)
                    for j in range(pieces):
                        N.check(lib.bb_copy_async(C.c_void_p(dst + j * piece), C.c_void_p(src + j * piece), piece,
                                                  C.c_void_p(s.cuda_stream)))
                for s in streams[:k]:
                    cur.wait_stream(s)
            e1.record(cur)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / 1e3], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            rates.append(n / float(t.item()) / 1e9)
        tag = ("_arena_dst" if arena_dst else "") + (f"_{pieces}pieces" if pieces > 1 else "")
        rates.sort()
        out[f"{kind}_{'bidir' if both else 'unidir'}_{k}streams{tag}_GBps_per_direction"] = {
            "best": rates[-1], "median": rates[len(rates) // 2], "worst": rates[0]}

    for kind in ("push", "pull"):
        for both in (False, True):
            for k in (1, 2):
                run(kind, both, k)
    for kind in ("push", "pull"):
        run(kind, True, 1, pieces=2)
    run("pull", True, 1, arena_dst=True)
    out["CUDA_DEVICE_MAX_CONNECTIONS"] = os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS")
    if rank == 0:
        print(json.dumps({"ipc_arena_copy_engine": out, "bytes_per_copy": n}), flush=True)
    ch.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
