"""Parity at the headline configuration itself (cfg3: 1M tokens, causal, zigzag, 32 heads,
d=128) on the production ring (ProcessRing, copy-engine transport, one process per GPU):
forward + burst backward over 4 GPUs, then sampled rows against float64 on the GPU -- O / lse /
dQ of 256 query rows and dK / dV of 256 key rows for two heads, the same reference and
tolerances as tests/test_scale_parity_gpu.py (cfg2 / cfg4 at full size on one GPU).

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 tools/parity_1m.py [--seq N]
Exits non-zero on a mismatch; used by tests/test_ring_multigpu.py when >= 4 GPUs are visible.
"""

import argparse
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2509_19836_b200 import masks as M  # noqa: E402
from paper_2509_19836_b200.partitioning import ShardLayout, device_token_ids  # noqa: E402
from paper_2509_19836_b200.ring import ProcessRing  # noqa: E402
from test_scale_parity_gpu import TOL_G, TOL_LSE, TOL_O, _fp64_reference  # noqa: E402

HEADS_CHECKED = (0, 21)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=1 << 20)
    ap.add_argument("--heads", type=int, default=32)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    n, h, d = args.seq, args.heads, 128
    layout = ShardLayout("zigzag", n, world)
    ids = torch.from_numpy(device_token_ids(layout, rank + 1) - 1).to(dev)  # shard row r holds token ids[r]

    def glob(seed):  # the same global tensor on every rank (same generator), head by head
        g = torch.Generator(device=dev).manual_seed(seed)
        return (torch.rand(n, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)

    shards, keep = [], []
    for seed in (1, 2, 3, 4):  # Q, K, V, dO
        t = glob(seed)
        shards.append(t.index_select(0, ids).contiguous())
        if rank == 0:
            keep.append(t[:, list(HEADS_CHECKED)].contiguous())
        del t
    torch.cuda.empty_cache()
    q, k, v, do = shards
    ring = ProcessRing(layout, M.causal_mask(), head_dim=d)
    o, lse = ring.forward(q, k, v)
    dq, dk, dv = ring.backward(q, k, v, do, o, lse)
    torch.cuda.synchronize()

    rng = np.random.default_rng(7)
    rows = np.unique(np.concatenate([[0, n - 1], rng.choice(n, 254, replace=False)]))
    cols = np.unique(np.concatenate([[0, n - 1], rng.choice(n, 254, replace=False)]))
    hsel = list(HEADS_CHECKED)
    # each rank contributes the sampled rows it owns (global row -> value, NaN elsewhere)
    inv = torch.full((n,), -1, dtype=torch.int64, device=dev)
    inv[ids] = torch.arange(ids.numel(), device=dev)

    def collect(t, which, per_head):  # t: [rows, H, d] or lse [H, rows]
        sel = torch.as_tensor(which, device=dev)
        loc = inv[sel]
        own = loc >= 0
        if per_head == "lse":
            out = torch.full((len(hsel), len(which)), float("nan"), dtype=torch.float64, device=dev)
            out[:, own] = t[hsel][:, loc[own]].double()
        else:
            out = torch.full((len(which), len(hsel), d), float("nan"), dtype=torch.float64, device=dev)
            out[own] = t[loc[own]][:, hsel].double()
        gathered = [torch.empty_like(out) for _ in range(world)]
        dist.all_gather(gathered, out)
        res = gathered[0]
        for x in gathered[1:]:
            res = torch.where(torch.isnan(res), x, res)
        return res

    got = {"o": collect(o, rows, None), "lse": collect(lse, rows, "lse"), "dq": collect(dq, rows, None),
           "dk": collect(dk, cols, None), "dv": collect(dv, cols, None)}
    ring.close()  # collective; free the ring's arenas and state before the float64 reference
    del q, k, v, do, o, lse, dq, dk, dv, shards, inv
    torch.cuda.empty_cache()
    failures = 0
    if rank == 0:
        qg, kg, vg, dog = keep
        ar_rows = rows
        for i, head in enumerate(hsel):
            ref = _fp64_reference(qg[:, i].double(), kg[:, i].double(), vg[:, i].double(), dog[:, i].double(),
                                  lambda qi, ki: ki[None, :] <= qi[:, None], lambda q0, q1: (0, q1),
                                  ar_rows, cols, 1 / math.sqrt(d), chunk=2048)
            checks = {
                "o": float((got["o"][:, i] - ref[0]).abs().max()),
                "lse": float((got["lse"][i] - ref[1]).abs().max()),
                "dq": float(torch.linalg.norm(got["dq"][:, i] - ref[2]) / torch.linalg.norm(ref[2])),
                "dk": float(torch.linalg.norm(got["dk"][:, i] - ref[3]) / torch.linalg.norm(ref[3])),
                "dv": float(torch.linalg.norm(got["dv"][:, i] - ref[4]) / torch.linalg.norm(ref[4])),
            }
            tol = {"o": TOL_O, "lse": TOL_LSE, "dq": TOL_G, "dk": TOL_G, "dv": TOL_G}
            bad = [kk for kk in checks if not checks[kk] < tol[kk]]
            failures += len(bad)
            print(f"seq {n} world {world} head {head}: " + ", ".join(f"{kk} {checks[kk]:.2e}" for kk in checks)
                  + (f"  FAIL {bad}" if bad else "  ok"), flush=True)
    t = torch.tensor([failures], device=dev)
    dist.all_reduce(t)
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
