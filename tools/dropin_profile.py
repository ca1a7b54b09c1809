"""Phase timing of the burstsim drop-in call sequence on one GPU (bench.py's e2e_dropin_api):
NumPy in -> make_device_states -> distributed_forward -> shard_rows(dO) -> burst_backward ->
backward_grads (float64 NumPy out).  Developer tool."""

import argparse
import time

import numpy as np
import torch

import paper_2509_19836_b200 as bb

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=131072)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--no-prefault", action="store_true")
args = ap.parse_args()
n, h, d = args.seq, args.heads, 128
layout = bb.ShardLayout("zigzag", n, 1)
mask = bb.causal_mask()
rng = np.random.default_rng(0)
q, k, v, do = (rng.uniform(-1, 1, (n, h, d)).astype(np.float32) for _ in range(4))


def phase(name, fn, times):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    times[name] = times.get(name, 0.0) + time.perf_counter() - t0
    return out


for rep in range(2):
    times = {}
    st = phase("make_device_states", lambda: bb.make_device_states(layout, q, k, v), times)
    phase("distributed_forward", lambda: bb.distributed_forward(st, layout, mask), times)
    dos = phase("shard_rows(dO)", lambda: bb.shard_rows(layout, do), times)
    phase("burst_backward", lambda: bb.burst_backward(st, dos, layout, mask), times)
    phase("backward_grads", lambda: bb.backward_grads(st), times)
    del st
    torch.cuda.empty_cache()
print({k2: round(v2, 3) for k2, v2 in times.items()}, "total", round(sum(times.values()), 3), flush=True)

# the same sequence without the per-phase synchronisation (as a caller runs it): host work in
# backward_grads (result allocation) overlaps the backward kernels.  --no-prefault: results
# allocated with a plain np.empty (first-touch page faults inside the copy)
import sys  # noqa: E402

from paper_2509_19836_b200 import hostio  # noqa: E402

if "--no-prefault" in sys.argv:
    hostio.empty_f64 = lambda t: np.empty(tuple(t.shape), dtype=np.float64)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = bb.make_device_states(layout, q, k, v)
    bb.distributed_forward(st, layout, mask)
    bb.burst_backward(st, bb.shard_rows(layout, do), layout, mask)
    t1 = time.perf_counter()
    g = bb.backward_grads(st)
    t2 = time.perf_counter()
    del st
    torch.cuda.empty_cache()
print({"unsynchronised_total": round(t2 - t0, 3), "backward_grads_call": round(t2 - t1, 3)}, flush=True)
