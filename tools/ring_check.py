"""Multi-GPU ring parity (torchrun, NCCL): ProcessRing with the sm_100a kernels vs the CPU oracle.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port 29511 tools/ring_check.py
Exits non-zero on mismatch.  Used by tests/test_ring_multigpu.py when >= 2 GPUs are visible.
"""

import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # see bench.py

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_19836_b200 import masks as M  # noqa: E402
from paper_2509_19836_b200.fabric import Topology  # noqa: E402
from paper_2509_19836_b200.partitioning import ShardLayout, device_token_ids  # noqa: E402
from paper_2509_19836_b200.ring import ProcessRing  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    opts = dist.ProcessGroupNCCL.Options()
    opts.is_high_priority_stream = True  # see bench.py: NCCL P2P CTAs must win free SMs
    dist.init_process_group("nccl", device_id=dev, pg_options=opts)
    from oracle import burst_oracle as O

    failures = 0
    n, d = 1024 * world, 128
    cases = [("zigzag", (1, world), "causal", 4, 4, "burst_backward"), ("zigzag", (1, world), "causal", 4, 2, "ring_backward")]
    if world == 4:
        cases.append(("striped", (2, 2), "window", 4, 4, "burst_backward"))
    for kind, topo, mname, hq, hkv, backward in cases:
        layout = ShardLayout(kind, n, world)
        mask = {"causal": M.causal_mask(), "window": M.sliding_window_mask(n // 3)}[mname]
        mt = {"causal": ("causal", None, None, None), "window": ("sliding_window", n // 3, None, None)}[mname]
        rng = np.random.default_rng(1)
        glob = [torch.from_numpy(rng.uniform(-1, 1, (n, h, d))).float().to(torch.bfloat16) for h in (hq, hkv, hkv, hq)]
        rows = torch.from_numpy(device_token_ids(layout, rank + 1) - 1)
        q, k, v, do = (t[rows].contiguous().to(dev) for t in glob)
        ref = O.mh_ring_attention(*(t.double().numpy() for t in glob), (kind, n, world, None), mt, O.ring_visit(*topo),
                                  backward="burst" if backward == "burst_backward" else "ring")
        r = rows.numpy()
        variants = [("ce", None), ("collective", None)] + ([("ce", 1)] if backward == "burst_backward" else [])
        if backward == "burst_backward" and topo[0] == 1:
            variants.append(("autograd", None))
        for transport, slots in variants:
            if transport == "autograd":  # BurstAttention.apply (CE ring) with sequence-selective recompute
                from paper_2509_19836_b200.autograd import BurstAttention
                from paper_2509_19836_b200.checkpointing import CheckpointPolicy

                ring = ProcessRing(layout, mask, Topology(*topo), head_dim=d)
                ql, kl, vl = (t.clone().requires_grad_() for t in (q, k, v))
                o, lse = BurstAttention.apply(ql, kl, vl, ring, backward, CheckpointPolicy("sequence_selective", 0.5))
                (o * do.float()).sum().backward()
                dq, dk, dv = ql.grad.float(), kl.grad.float(), vl.grad.float()
                o, lse = o.detach(), lse.detach()
            else:
                ring = ProcessRing(layout, mask, Topology(*topo), head_dim=d, transport=transport, slots=slots)
                for rep in range(2):  # later passes exercise the cross-pass slot hand-over (flag epochs)
                    traced = transport == "ce" and rep == 1
                    if traced:  # measured timeline of the second pass (validated on assembly)
                        ring.trace_begin()
                    o16 = torch.empty(q.shape, dtype=torch.bfloat16, device=dev)
                    o, lse = ring.forward(q, k, v, o16=o16)
                    if not torch.equal(o16, o.to(torch.bfloat16)):  # bf16 O from the last step's epilogue
                        print(f"rank {rank} FAIL bf16 O copy differs from bf16(O)", flush=True)
                        failures += 1
                    dq, dk, dv = ring.backward(q, k, v, do, o, lse, kind=backward)
                    if traced:
                        tl = ring.trace_collect()
                        if not tl.by_kind("compute") or not (tl.by_kind("send_intra") or tl.by_kind("send_inter")):
                            print(f"rank {rank} FAIL timeline without kernels or pushes", flush=True)
                            failures += 1
            torch.cuda.synchronize()
            ring.close()  # collective: frees the copy-engine arenas after every rank's passes
            failures += _report(rank, f"{kind} {topo} {mname} {backward} {transport} slots={slots}", o, lse, dq, dk, dv,
                                ref, r, ring.stats.bytes_sent)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(1 if failures else 0)


def _report(rank, label, o, lse, dq, dk, dv, ref, r, sent) -> int:
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    errs = {
        "o": float(np.abs(o.double().cpu().numpy() - ref["o"][r]).max()),
        "lse": float(np.abs(lse.double().cpu().numpy() - ref["lse"][:, r]).max()),
        "dq": rel(dq.double().cpu().numpy(), ref["dq"][r]),
        "dk": rel(dk.double().cpu().numpy(), ref["dk"][r]),
        "dv": rel(dv.double().cpu().numpy(), ref["dv"][r]),
    }
    ok = errs["o"] < 1e-2 and errs["lse"] < 2e-3 and errs["dq"] < 1e-2 and errs["dk"] < 1e-2 and errs["dv"] < 1e-2
    line = f"rank {rank} {label}: {'ok' if ok else 'FAIL'} {errs} sent={sent}"
    print(line, flush=True)
    with open(os.path.join(os.environ.get("BB_RING_LOG_DIR", "."), f"ring_check_rank{rank}.log"), "a") as f:
        f.write(line + "\n")
    return int(not ok)


if __name__ == "__main__":
    main()
