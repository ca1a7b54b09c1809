"""One-process-per-GPU BurstAttention ring over torch.distributed (NCCL / NVLink).

This is the multi-GPU production path (torchrun, rank r = ring device r+1).
Each rank owns one shard of Q/K/V/dO (bf16 [n, H, d]) resident in HBM and runs
the same sm_100a kernels as the single-process engine; what moves between ranks
is exactly the reference's payloads (distributed.py:64-101):

  forward        K_j, V_j                               (KvPayload)
  burst backward Q_j, dO_j, D_j, lse_j  +  dQ_j partial  (QPayload)
  ring backward  K_j, V_j               +  dK_j/dV_j partials (KvPayload + grads)

Overlap: the read-only part of step t+1's payload is posted
(NCCL send/recv on NCCL's stream) before step t's kernel is launched, so the
transfer runs under the compute; gradient partials are produced into a fresh
buffer by step t's kernel and sent straight to their owner afterwards (delayed
gradient send) while step t+1 computes.  Own shard is computed first, so a
pass needs G-1 read-only hops (the reference's MessageLog still counts G).
The visit order follows ``build_ring_plan``: flat (1xG) receives from the ring
predecessor; a two-level plan (e.g. 2x4) orders shards node-major with intra
hops inside a node and one inter hop per round.  Inside an NVSwitch box every
hop is one NVLink traversal, so both are the same bandwidth class.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from . import kernels as K
from .fabric import BURST_BACKWARD, FORWARD, RING_BACKWARD, Topology, build_ring_plan, single_node_topology
from .masks import MaskSpec, validate_mask
from .partitioning import ShardLayout, pair_count_matrix


def ring_schedule(topology: Topology, rank: int) -> list[int]:
    """0-based shard order this rank computes: own first, then the plan's arrival order."""
    plan = build_ring_plan(topology)
    order = list(plan.visit[rank])
    order.remove(rank)
    return [rank] + order


@dataclass
class RingStats:
    bytes_sent: int = 0
    launches: int = 0
    kernel_events: list = field(default_factory=list)  # (start, end) CUDA events when recording


class ProcessRing:
    """Ring attention for one rank: ``forward`` -> (O, lse); ``backward`` -> (dQ, dK, dV)."""

    def __init__(self, layout: ShardLayout, mask: MaskSpec, topology: Topology | None = None, group=None, head_dim: int | None = None):
        self.layout = layout
        self.mask = mask
        validate_mask(mask, layout.seq_len)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if self.world != layout.devices:
            raise ValueError(f"world size {self.world} != layout devices {layout.devices}")
        self.topology = topology if topology is not None else single_node_topology(layout.devices)
        if self.topology.total_devices != layout.devices:
            raise ValueError(f"topology has {self.topology.total_devices} devices but layout shards {layout.devices}")
        self.order = ring_schedule(self.topology, self.rank)
        self.counts = pair_count_matrix(layout, mask)  # [query dev, key dev] allowed pairs
        self.device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
        self.dmask = K.device_mask(mask, self.device)  # (host-side tests swap K for a CPU double)
        self.head_dim = head_dim
        self.stats = RingStats()
        self.compute = True  # False: run only the exchanges (communication-alone timing)
        self.record = False  # True: CUDA events around every kernel launch (compute-lane time)

    def _launch(self, fn, *a, **kw):
        if not self.compute:
            return
        if self.record:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(*a, **kw)
            e1.record()
            self.stats.kernel_events.append((e0, e1))
        else:
            fn(*a, **kw)
        self.stats.launches += 1

    def kernel_seconds(self) -> float:
        """Sum of recorded kernel durations (call after synchronizing)."""
        return sum(a.elapsed_time(b) for a, b in self.stats.kernel_events) / 1e3

    # -------------------------------------------------------------- helpers
    def _peer(self, t: int) -> tuple[int, int]:
        """(rank that receives my step-t payload, rank I receive from) for step t >= 1: the shard
        order is a rotation, so at step t I hold shard order[t] and need it from its owner's path;
        with NVSwitch the payload is fetched straight from its owner."""
        src = self.order[t]
        # who needs MY shard at step t: the rank whose order[t] == me
        dst = next(r for r in range(self.world) if ring_schedule(self.topology, r)[t] == self.rank)
        return dst, src

    def _exchange(self, send: list[torch.Tensor], recv: list[torch.Tensor], dst: int, src: int):
        ops = [dist.P2POp(dist.isend, t, dst, self.group) for t in send]
        ops += [dist.P2POp(dist.irecv, t, src, self.group) for t in recv]
        self.stats.bytes_sent += sum(t.numel() * t.element_size() for t in send)
        return dist.batch_isend_irecv(ops)

    def _scale(self, d_pad: int) -> float:
        return 1.0 / math.sqrt(self.head_dim or d_pad)

    # -------------------------------------------------------------- forward
    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor | None = None,
                lse: torch.Tensor | None = None, n_q: int | None = None):
        """Ring forward.  ``n_q`` < n runs only the first n_q query rows (the rows a
        sequence-selective checkpoint dropped, see ``recompute``); K/V still circulate whole."""
        n, hq, d = q.shape
        if n_q is not None and n_q < n:
            o_full = torch.zeros(n, hq, d, dtype=torch.float32, device=q.device) if o is None else o
            lse_full = torch.full((hq, n), float("-inf"), device=q.device) if lse is None else lse
            saved = self.compute
            self.compute = saved and n_q > 0  # the exchanges are collective: always run them
            try:
                o_p, lse_p = self.forward(q[:n_q].contiguous(), k, v, o_full[:n_q], None)
            finally:
                self.compute = saved
            lse_full[:, :n_q].copy_(lse_p)
            return o_full, lse_full
        o = torch.zeros(n, hq, d, dtype=torch.float32, device=q.device) if o is None else o.zero_()
        lse = torch.full((hq, n), float("-inf"), device=q.device) if lse is None else lse.fill_(float("-inf"))
        bufs = [(k, v)] + [(torch.empty_like(k), torch.empty_like(v)) for _ in range(2)]
        pending = None
        for t in range(self.world):
            j = self.order[t]
            kv = bufs[0] if t == 0 else bufs[1 + (t - 1) % 2]
            if pending is not None:
                for w in pending:
                    w.wait()
                pending = None
            if t + 1 < self.world:  # post step t+1's K/V before launching step t's kernel
                dst, src = self._peer(t + 1)
                nxt = bufs[1 + t % 2]
                pending = self._exchange([k, v], list(nxt), dst, src)
            if self.counts[self.rank, j]:
                self._launch(K.attn_fwd_step, q, kv[0], kv[1], o, lse, self.layout, self.dmask, self.rank + 1, j + 1,
                             self._scale(d), n_q=q.shape[0])
        return o, lse

    def recompute(self, q, k, v, o, lse, policy) -> int:
        """Sequence-selective checkpointing (checkpointing.py:141-157): recompute (O, lse) for this
        rank's rows with global token id <= boundary -- a prefix of the shard -- with the ring
        forward restricted to them.  Returns the number of recomputed rows."""
        from .checkpointing import _prefix_rows

        p = _prefix_rows(self.layout, policy.stored_from(self.layout.seq_len))[self.rank]
        self.forward(q, k, v, o, lse, n_q=p)  # collective: every rank takes part, p may be 0
        return p

    # -------------------------------------------------------------- backward
    def backward(self, q, k, v, do, o, lse, kind: str = BURST_BACKWARD, dq=None, dk=None, dv=None):
        """Gradients of sum(O * dO); ``kind`` picks the payload that circulates."""
        n, hq, d = q.shape
        delta = torch.empty_like(lse)
        self._launch(K.bwd_preprocess, do, o, delta)
        dq = torch.zeros(q.shape, dtype=torch.float32, device=q.device) if dq is None else dq.zero_()
        dk = torch.zeros(k.shape, dtype=torch.float32, device=q.device) if dk is None else dk.zero_()
        dv = torch.zeros(v.shape, dtype=torch.float32, device=q.device) if dv is None else dv.zero_()
        if kind == BURST_BACKWARD:
            self._burst(q, k, v, do, lse, delta, dq, dk, dv, d)
        elif kind == RING_BACKWARD:
            self._ringbwd(q, k, v, do, lse, delta, dq, dk, dv, d)
        else:
            raise ValueError(f"unknown backward {kind!r}")
        return dq, dk, dv

    def _burst(self, q, k, v, do, lse, delta, dq, dk, dv, d):
        own = (q, do, lse, delta)
        bufs = [own] + [tuple(torch.empty_like(x) for x in own) for _ in range(2)]
        parts = [torch.empty_like(dq) for _ in range(2)]
        inbox = [torch.empty_like(dq) for _ in range(2)]
        pending = None
        grad_pending = None
        for t in range(self.world):
            j = self.order[t]
            payload = bufs[0] if t == 0 else bufs[1 + (t - 1) % 2]
            if pending is not None:
                for w in pending:
                    w.wait()
                pending = None
            if t + 1 < self.world:
                dst, src = self._peer(t + 1)
                pending = self._exchange(list(own), list(bufs[1 + t % 2]), dst, src)
            if t == 0:
                acc = dq  # own shard: accumulate in place
            else:
                acc = parts[t % 2]
                if grad_pending is not None and grad_pending[1] is acc:
                    for w in grad_pending[0]:
                        w.wait()
                    dq.add_(grad_pending[2])
                    grad_pending = None
                acc.zero_()
            if self.counts[j, self.rank]:
                self._launch(K.attn_bwd_step, payload[0], k, v, payload[1], payload[2], payload[3], acc, dk, dv,
                             self.layout, self.dmask, j + 1, self.rank + 1, self._scale(d))
            if t > 0:  # delayed gradient send: my partial for shard j goes to its owner j;
                # I receive the partial for MY shard from the rank that computed it at step t
                if grad_pending is not None:
                    for w in grad_pending[0]:
                        w.wait()
                    dq.add_(grad_pending[2])
                box = inbox[t % 2]
                works = self._exchange([acc], [box], j, self._who_had_me(t))
                grad_pending = (works, acc, box)
        if grad_pending is not None:
            for w in grad_pending[0]:
                w.wait()
            dq.add_(grad_pending[2])

    def _ringbwd(self, q, k, v, do, lse, delta, dq, dk, dv, d):
        own = (k, v)
        bufs = [own] + [tuple(torch.empty_like(x) for x in own) for _ in range(2)]
        parts = [(torch.empty_like(dk), torch.empty_like(dv)) for _ in range(2)]
        inbox = [(torch.empty_like(dk), torch.empty_like(dv)) for _ in range(2)]
        pending = None
        grad_pending = None
        for t in range(self.world):
            j = self.order[t]
            kv = bufs[0] if t == 0 else bufs[1 + (t - 1) % 2]
            if pending is not None:
                for w in pending:
                    w.wait()
                pending = None
            if t + 1 < self.world:
                dst, src = self._peer(t + 1)
                pending = self._exchange(list(own), list(bufs[1 + t % 2]), dst, src)
            if t == 0:
                acc = (dk, dv)
            else:
                acc = parts[t % 2]
                if grad_pending is not None and grad_pending[1] is acc:
                    for w in grad_pending[0]:
                        w.wait()
                    dk.add_(grad_pending[2][0])
                    dv.add_(grad_pending[2][1])
                    grad_pending = None
                acc[0].zero_()
                acc[1].zero_()
            if self.counts[self.rank, j]:
                self._launch(K.attn_bwd_step, q, kv[0], kv[1], do, lse, delta, dq, acc[0], acc[1],
                             self.layout, self.dmask, self.rank + 1, j + 1, self._scale(d))
            if t > 0:
                if grad_pending is not None:
                    for w in grad_pending[0]:
                        w.wait()
                    dk.add_(grad_pending[2][0])
                    dv.add_(grad_pending[2][1])
                box = inbox[t % 2]
                works = self._exchange(list(acc), list(box), j, self._who_had_me(t))
                grad_pending = (works, acc, box)
        if grad_pending is not None:
            for w in grad_pending[0]:
                w.wait()
            dk.add_(grad_pending[2][0])
            dv.add_(grad_pending[2][1])

    def _who_had_me(self, t: int) -> int:
        """Rank that computed on MY shard at step t (it sends me that gradient partial)."""
        return next(r for r in range(self.world) if ring_schedule(self.topology, r)[t] == self.rank)


def pass_flops(layout: ShardLayout, mask: MaskSpec, heads: int, head_dim: int) -> tuple[float, float]:
    """Algorithmic FLOPs of the whole job: forward 4*d*H*P, backward 10*d*H*P (FlashAttention
    convention incl. the S recompute; P = exact unmasked pairs)."""
    from .masks import unmasked_pair_count

    p = unmasked_pair_count(mask, layout.seq_len)
    return 4.0 * head_dim * heads * p, 10.0 * head_dim * heads * p
