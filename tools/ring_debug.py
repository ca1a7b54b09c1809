"""Watchdog run of one CE ring pass pair (torchrun): polls the streams instead of blocking, and
on a stall dumps every channel's flag words (read on a private stream) and which phase is stuck.

    torchrun --nproc-per-node N tools/ring_debug.py [burst_backward|ring_backward] [hq] [hkv]
"""

import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_19836_b200 import masks as M  # noqa: E402
from paper_2509_19836_b200.fabric import Topology  # noqa: E402
from paper_2509_19836_b200.partitioning import ShardLayout  # noqa: E402
from paper_2509_19836_b200.ring import ProcessRing  # noqa: E402


def dump(ring, rank):
    s = torch.cuda.Stream(priority=0)
    out = []
    for name, ch in ring._channels.items():
        w = ch.world
        flags = ch.arena[ch.flags_off: ch.flags_off + 8 * w]
        host = torch.empty(8 * w, dtype=torch.uint8, pin_memory=True)
        with torch.cuda.stream(s):
            host.copy_(flags, non_blocking=True)
        deadline = time.time() + 5
        while not s.query() and time.time() < deadline:
            time.sleep(0.01)
        v = host.view(torch.int32).tolist() if s.query() else "copy blocked"
        out.append(f"{name}: epoch={ch.epoch} ready={v[:w] if isinstance(v, list) else v} free={v[w:] if isinstance(v, list) else ''}")
    return f"rank {rank} " + " | ".join(out)


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "ring_backward"
    hq = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    hkv = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    n, d = 1024 * world, 128
    layout = ShardLayout("zigzag", n, world)
    ring = ProcessRing(layout, M.causal_mask(), Topology(1, world), head_dim=d, transport="ce")
    g = torch.Generator(device=dev).manual_seed(rank)
    rnd = lambda h: (torch.rand(n // world, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)  # noqa: E731
    q, k, v, do = rnd(hq), rnd(hkv), rnd(hkv), rnd(hq)
    ok = True
    for rep in range(3):
        for phase in ("forward", "backward"):
            t0 = time.time()
            if phase == "forward":
                o, lse = ring.forward(q, k, v)
            else:
                ring.backward(q, k, v, do, o, lse, kind=kind)
            ev = torch.cuda.Event()
            ev.record()
            while not ev.query():
                if time.time() - t0 > 30:
                    print(f"rank {rank} STALL rep {rep} {phase}: " + dump(ring, rank), flush=True)
                    ok = False
                    break
                time.sleep(0.01)
            if not ok:
                break
            print(f"rank {rank} rep {rep} {phase} done {time.time() - t0:.3f}s " + dump(ring, rank), flush=True)
        if not ok:
            break
    sys.stdout.flush()
    os._exit(0 if ok else 1)


if __name__ == "__main__":
    main()
