"""Multi-process ring host logic on CPU (gloo, world sizes 2, 4 and 8).

ProcessRing's schedule -- which shard each rank computes at each step, who sends
it, and where every gradient partial goes -- is exercised for real over
torch.distributed (gloo) with the sm_100a kernels swapped for a float64 CPU test
double of the same step semantics.  Gathered results must equal the CPU oracle
(the reference algorithm); the kernel math itself is covered by the GPU suites.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import burst_oracle as O


class FakeKernels:
    """CPU double of paper_2509_19836_b200.kernels for one (query shard, key shard) step."""

    def __init__(self, layout, mask_tuple):
        from paper_2509_19836_b200.partitioning import device_token_ids

        self.ids = lambda dev: device_token_ids(layout, dev)
        self.mask = mask_tuple

    def device_mask(self, mask, device):
        return None

    def _allowed(self, qdev, kdev, nq, nk):
        a = O.allowed(self.mask, self.ids(qdev)[:nq], self.ids(kdev)[:nk])
        return torch.from_numpy(a)

    def attn_fwd_step(self, q, k, v, o, lse, layout, dmask, qdev, kdev, scale, n_q=None, o_bf16=None):
        nq, nk = q.shape[0], k.shape[0]
        rep = q.shape[1] // k.shape[1]
        am = self._allowed(qdev, kdev, nq, nk)
        kr, vr = k.repeat_interleave(rep, 1), v.repeat_interleave(rep, 1)
        s = torch.einsum("qhd,khd->hqk", q, kr) * scale
        s = s.masked_fill(~am[None], float("-inf"))
        l_step = torch.logsumexp(s, -1)
        p = torch.exp(s - l_step[..., None]).nan_to_num(0.0)
        o_step = torch.einsum("hqk,khd->qhd", p, vr)
        l_new = torch.logaddexp(lse, l_step)
        w_s = torch.exp(l_step - l_new).nan_to_num(0.0).t()[..., None]
        w_o = torch.exp(lse - l_new).nan_to_num(0.0).t()[..., None]
        o.copy_(w_s * o_step + w_o * o)
        lse.copy_(l_new)
        if o_bf16 is not None:  # (a float32 stand-in for the bf16 copy: the fakes run in float64)
            o_bf16.copy_(o)

    def bwd_preprocess(self, do, o, delta):
        delta.copy_((do * o).sum(-1).t())

    def fill_(self, t, value=0.0):
        return t.fill_(value)

    def add_rows_(self, dst, src):
        return dst.add_(src)

    def attn_bwd_step(self, q, k, v, do, lse, delta, dq, dk, dv, layout, dmask, qdev, kdev, scale):
        rep = q.shape[1] // k.shape[1]
        am = self._allowed(qdev, kdev, q.shape[0], k.shape[0])
        kr, vr = k.repeat_interleave(rep, 1), v.repeat_interleave(rep, 1)
        s = torch.einsum("qhd,khd->hqk", q, kr) * scale
        s = s.masked_fill(~am[None], float("-inf"))
        p = torch.exp(s - lse[..., None]).nan_to_num(0.0)
        dp = torch.einsum("qhd,khd->hqk", do, vr)
        ds = p * (dp - delta[..., None])
        dq += torch.einsum("hqk,khd->qhd", ds, kr) * scale
        dk_h = torch.einsum("hqk,qhd->khd", ds, q) * scale
        dv_h = torch.einsum("hqk,qhd->khd", p, do)
        dk += dk_h.reshape(dk_h.shape[0], k.shape[1], rep, -1).sum(2)
        dv += dv_h.reshape(dv_h.shape[0], k.shape[1], rep, -1).sum(2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_19836_b200 import masks as M
        from paper_2509_19836_b200 import ring as R
        from paper_2509_19836_b200.fabric import Topology
        from paper_2509_19836_b200.partitioning import ShardLayout, device_token_ids

        kind, n, topo, mname, hq, hkv, d, backward = case
        layout = ShardLayout(kind, n, world)
        mask = {"causal": M.causal_mask(), "full": M.full_mask(), "window": M.sliding_window_mask(n // 3)}[mname]
        mtuple = {"causal": ("causal", None, None, None), "full": ("full", None, None, None),
                  "window": ("sliding_window", n // 3, None, None)}[mname]
        R.K = FakeKernels(layout, mtuple)
        rng = np.random.default_rng(0)
        q, k, v, do = (torch.from_numpy(rng.uniform(-1, 1, (n, h, d))) for h in (hq, hkv, hkv, hq))
        rows = torch.from_numpy(device_token_ids(layout, rank + 1) - 1)
        ring = R.ProcessRing(layout, mask, Topology(*topo), head_dim=d)
        o16 = torch.full((rows.shape[0], hq, d), float("nan"), dtype=torch.float32)
        o, lse = ring.forward(q[rows].contiguous(), k[rows].contiguous(), v[rows].contiguous(), o16=o16)
        assert torch.equal(o16, o.float())  # the last launched step leaves the copy of the final O
        dq, dk, dv = ring.backward(q[rows].contiguous(), k[rows].contiguous(), v[rows].contiguous(),
                                   do[rows].contiguous(), o, lse, kind=backward)
        # sequence-selective checkpoint: drop (O, lse) of rows with id <= N/2, recompute them
        from paper_2509_19836_b200.checkpointing import CheckpointPolicy

        o2, lse2 = o.clone(), lse.clone()
        o2.zero_()
        lse2.fill_(float("nan"))
        pol = CheckpointPolicy("sequence_selective", 0.5)
        p_rows = ring.recompute(q[rows].contiguous(), k[rows].contiguous(), v[rows].contiguous(), o2, lse2, pol)
        ids = device_token_ids(layout, rank + 1)
        assert p_rows == int((ids <= n // 2).sum())
        assert torch.allclose(o2[:p_rows], o[:p_rows]) and torch.allclose(lse2[:, :p_rows], lse[:, :p_rows])
        out_q.put((rank, rows.numpy(), o.numpy(), lse.numpy(), dq.numpy(), dk.numpy(), dv.numpy(), ring.stats.bytes_sent))
    finally:
        dist.destroy_process_group()


CASES = [
    ("zigzag", 32, (1, 2), "causal", 2, 2, 8, "burst_backward"),
    ("zigzag", 32, (1, 2), "causal", 2, 1, 8, "ring_backward"),
    ("zigzag", 64, (1, 4), "causal", 2, 2, 8, "burst_backward"),
    ("striped", 64, (2, 2), "window", 4, 2, 8, "burst_backward"),
    ("contiguous", 64, (2, 2), "full", 2, 2, 4, "ring_backward"),
    # the driver's 8-GPU scaling run: flat 1x8 and two-level 2x4 plans
    ("zigzag", 128, (1, 8), "causal", 2, 2, 8, "burst_backward"),
    ("striped", 128, (2, 4), "window", 2, 1, 8, "ring_backward"),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[1]}-{c[2][0]}x{c[2][1]}-{c[3]}-{c[7]}")
def test_process_ring_matches_oracle(case):
    kind, n, topo, mname, hq, hkv, d, backward = case
    world = topo[0] * topo[1]
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [out_q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(0)
    q, k, v, do = (rng.uniform(-1, 1, (n, h, d)) for h in (hq, hkv, hkv, hq))
    mtuple = {"causal": ("causal", None, None, None), "full": ("full", None, None, None),
              "window": ("sliding_window", n // 3, None, None)}[mname]
    ref = O.mh_ring_attention(q, k, v, do, (kind, n, world, None), mtuple, O.ring_visit(*topo),
                              backward="burst" if backward == "burst_backward" else "ring")
    for rank, rows, o, lse, dq, dk, dv, sent in res:
        assert np.max(np.abs(o - ref["o"][rows])) < 2e-6  # fp32 accumulators (the product allocates O, lse, dQ, dK, dV in fp32)
        assert np.max(np.abs(lse - ref["lse"][:, rows])) < 2e-6  # fp32 accumulators (the product allocates O, lse, dQ, dK, dV in fp32)
        assert np.max(np.abs(dq - ref["dq"][rows])) < 2e-6  # fp32 accumulators (the product allocates O, lse, dQ, dK, dV in fp32)
        assert np.max(np.abs(dk - ref["dk"][rows])) < 2e-6  # fp32 accumulators (the product allocates O, lse, dQ, dK, dV in fp32)
        assert np.max(np.abs(dv - ref["dv"][rows])) < 2e-6  # fp32 accumulators (the product allocates O, lse, dQ, dK, dV in fp32)
        assert sent > 0  # own shard first: G-1 read-only hops per pass plus gradient partials


def _autograd_worker(rank, world, port, policy_frac, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_19836_b200 import masks as M
        from paper_2509_19836_b200 import ring as R
        from paper_2509_19836_b200.autograd import burst_attention
        from paper_2509_19836_b200.checkpointing import CheckpointPolicy
        from paper_2509_19836_b200.fabric import Topology
        from paper_2509_19836_b200.partitioning import ShardLayout, device_token_ids

        n, hq, hkv, d = 32, 2, 1, 8
        layout = ShardLayout("zigzag", n, world)
        R.K = FakeKernels(layout, ("causal", None, None, None))
        rng = np.random.default_rng(0)
        q, k, v, do = (torch.from_numpy(rng.uniform(-1, 1, (n, h, d))) for h in (hq, hkv, hkv, hq))
        rows = torch.from_numpy(device_token_ids(layout, rank + 1) - 1)
        ql, kl, vl = (t[rows].contiguous().requires_grad_() for t in (q, k, v))
        ring = R.ProcessRing(layout, M.causal_mask(), Topology(1, world), head_dim=d)
        policy = CheckpointPolicy("sequence_selective", policy_frac) if policy_frac is not None else None
        o = burst_attention(ql, kl, vl, ring, "burst_backward", policy)
        (o.double() * do[rows]).sum().backward()
        out_q.put((rank, rows.numpy(), o.detach().numpy(), ql.grad.numpy(), kl.grad.numpy(), vl.grad.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("policy_frac", [None, 0.5])
def test_autograd_function_matches_oracle(policy_frac):
    """BurstAttention.apply over a 2-rank gloo ring: O and the autograd gradients equal the
    oracle; with a sequence_selective policy the dropped (O, lse) prefix is recomputed."""
    world = 2
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_autograd_worker, args=(r, world, port, policy_frac, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [out_q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, hq, hkv, d = 32, 2, 1, 8
    rng = np.random.default_rng(0)
    q, k, v, do = (rng.uniform(-1, 1, (n, h, d)) for h in (hq, hkv, hkv, hq))
    ref = O.mh_ring_attention(q, k, v, do, ("zigzag", n, world, None), ("causal", None, None, None),
                              O.ring_visit(1, world), backward="burst")
    for rank, rows, o, dq, dk, dv in res:
        assert np.max(np.abs(o - ref["o"][rows])) < 2e-6
        assert np.max(np.abs(dq - ref["dq"][rows])) < 2e-6
        assert np.max(np.abs(dk - ref["dk"][rows])) < 2e-6
        assert np.max(np.abs(dv - ref["dv"][rows])) < 2e-6


def test_measured_events_assemble_into_a_valid_timeline():
    """ProcessRing.trace_collect's assembly (ring.assemble_timeline): per-rank kernel and push
    events become the reference's Timeline schema (fabric.py:366-388); pushes are split into
    intra / inter sends by the R x M topology and mirrored as the receiver's recv; the result
    passes validate_timeline, and an overlapping compute lane is rejected."""
    from paper_2509_19836_b200.fabric import Topology
    from paper_2509_19836_b200.ring import assemble_timeline

    per_rank = [
        [("compute", 0.0, 1.0, "fwd own", None), ("send", 0.1, 0.2, "kv step 1 1->2", 1),
         ("compute", 1.0, 2.0, "fwd k2", None)],
        [("compute", 0.0, 1.1, "fwd own", None), ("send", 0.1, 0.25, "kv step 1 2->1", 0),
         ("send", 0.3, 0.4, "kv step 2 2->3", 2)],
        [("compute", 0.0, 0.9, "fwd own", None)],
        [("compute", 0.0, 0.95, "fwd own", None), ("send", 0.5, 2.5, "dq step 1 4->1", 0)],
    ]
    tl = assemble_timeline(per_rank, Topology(2, 2))
    assert tl.makespan == 2.5
    kinds = {(e.device, e.kind, e.label) for e in tl.events}
    assert (1, "send_intra", "kv step 1 1->2") in kinds and (2, "recv", "recv kv step 1 1->2") in kinds
    assert (2, "send_inter", "kv step 2 2->3") in kinds and (3, "recv", "recv kv step 2 2->3") in kinds
    assert (4, "send_inter", "dq step 1 4->1") in kinds and (1, "recv", "recv dq step 1 4->1") in kinds
    per_rank[0].append(("compute", 1.5, 1.8, "overlapping", None))
    with pytest.raises(ValueError, match="compute lane overlaps"):
        assemble_timeline(per_rank, Topology(2, 2))
