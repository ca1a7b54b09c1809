"""Where the N>1 step spends time outside the attention kernels: one traced fwd + burst bwd
step of the bench's cfg2 workload, every rank's kernel and push events printed in order with
the idle gaps of the compute lane.  Developer tool (bench.py is the contract).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/ring_gaps.py [--seq 131072]
"""

import argparse
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_19836_b200 import masks as M  # noqa: E402
from paper_2509_19836_b200.partitioning import ShardLayout  # noqa: E402
from paper_2509_19836_b200.ring import ProcessRing  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=131072)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--comm-only", action="store_true", help="trace the exchanges with the kernels off")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    layout = ShardLayout("zigzag", args.seq, world)
    n, h, d = layout.shard_size, args.heads, 128
    g = torch.Generator(device=dev).manual_seed(rank)
    q, k, v, do = ((torch.rand(n, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(4))
    o = torch.empty(n, h, d, device=dev)
    lse = torch.empty(h, n, device=dev)
    dq, dk, dv = (torch.empty(n, h, d, device=dev) for _ in range(3))
    ring = ProcessRing(layout, M.causal_mask(), head_dim=d)

    def step():
        ring.forward(q, k, v, o, lse)
        ring.backward(q, k, v, do, o, lse, dq=dq, dk=dk, dv=dv)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    ring.compute = not args.comm_only
    ring.trace_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step()
    e1.record()
    tl = ring.trace_collect()
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1)
    from paper_2509_19836_b200.partitioning import pair_count_matrix

    counts = pair_count_matrix(layout, M.causal_mask())

    def rate(e, r):  # TFLOP/s of one traced attention launch (labels name the shard pair)
        import re
        lab = e.label
        m = re.match(r"forward q(\d+) x k(\d+)", lab)
        if m:
            i, j = int(m.group(1)) - 1, int(m.group(2)) - 1
            return 4.0 * d * h * counts[i, j] / (e.end - e.start) / 1e12
        m = re.match(r"dq shard (\d+) on (\d+)", lab)
        if m:
            i, j = int(m.group(1)) - 1, int(m.group(2)) - 1
            return 10.0 * d * h * counts[i, j] / (e.end - e.start) / 1e12
        m = re.match(r"dq own shard ([AB])", lab)
        if m:
            return 10.0 * d * h * counts[r, r] / 2 / (e.end - e.start) / 1e12
        return None

    if rank == 0:
        for r in range(world):
            evs = sorted(tl.device_events(r + 1), key=lambda e: e.start)
            comp = [e for e in evs if e.kind == "compute"]
            busy = sum(e.end - e.start for e in comp) * 1e3
            print(f"== rank {r}: step {step_ms:.2f} ms (rank 0 clock), kernels {busy:.2f} ms")
            prev_end = None
            for e in evs:
                gap = ""
                if e.kind == "compute":
                    if prev_end is not None and e.start - prev_end > 20e-6:
                        gap = f"   <- compute idle {1e3 * (e.start - prev_end):.3f} ms"
                    prev_end = e.end
                tf = rate(e, r) if e.kind == "compute" else None
                tfs = f"  [{tf:.0f} TF/s]" if tf else ""
                print(f"  {e.kind:11s} {1e3 * e.start:9.3f} {1e3 * e.end:9.3f} {1e3 * (e.end - e.start):8.3f}  {e.label}{tfs}{gap}")
    ring.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
