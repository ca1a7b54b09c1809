"""One-process-per-GPU BurstAttention ring over torch.distributed (NCCL / NVLink).

This is the multi-GPU production path (torchrun, rank r = ring device r+1).
Each rank owns one shard of Q/K/V/dO (bf16 [n, H, d]) resident in HBM and runs
the same sm_100a kernels as the single-process engine; what moves between ranks
is exactly the reference's payloads (distributed.py:64-101):

  forward        K_j, V_j                               (KvPayload)
  burst backward Q_j, dO_j, D_j, lse_j  +  dQ_j partial  (QPayload)
  ring backward  K_j, V_j               +  dK_j/dV_j partials (KvPayload + grads)

Two transports carry the payloads:

* ``"ce"`` (default on GPUs): copy-engine pushes over NVLink into CUDA-IPC
  arenas with stream-ordered flags (``peer.Channel``).  Every read-only payload
  of the pass is pushed at pass start on a copy stream, the consumer stream
  waits on a local flag right before the kernel that reads it, and gradient
  partials are pushed to their owner as soon as the kernel producing them ends
  (delayed gradient send).  No SM is used by the exchange, so the
  attention kernels, which hold every SM, never delay it.
* ``"collective"``: torch.distributed P2P (NCCL on GPUs, gloo for the CPU tests):
  the read-only part of step t+1's payload is posted before step t's kernel
  is launched; gradient partials are sent after the kernel.
  Own shard is computed first, so a
pass needs G-1 read-only hops (the reference's MessageLog still counts G).
The visit order follows ``build_ring_plan``: flat (1xG) receives from the ring
predecessor; a two-level plan (e.g. 2x4) orders shards node-major with intra
hops inside a node and one inter hop per round.  Inside an NVSwitch box every
hop is one NVLink traversal, so both are the same bandwidth class.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from . import kernels as K
from .fabric import (
    BURST_BACKWARD,
    FORWARD,
    RING_BACKWARD,
    Timeline,
    TimelineEvent,
    Topology,
    build_ring_plan,
    single_node_topology,
    validate_timeline,
)
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


def assemble_timeline(per_rank: list[list[tuple]], topology: Topology) -> Timeline:
    """Measured events of every rank -> the reference's Timeline schema (fabric.py:366-388).

    ``per_rank[r]`` holds (kind, start_s, end_s, label, peer) tuples of rank r on a common time
    base: kind "compute" (a kernel on the compute stream) or "send" (a copy-engine push to rank
    ``peer``).  A send becomes send_intra / send_inter by whether the two ranks share a node of
    the R x M topology, and is mirrored as the receiver's "recv <label>" over the same interval
    (the push lands in the receiver's arena while it runs), so validate_timeline's send/recv
    matching holds by construction and its compute-lane check tests the real launches."""
    m = topology.gpus_per_node
    evs = []
    for r, events in enumerate(per_rank):
        for kind, a, b, label, peer in events:
            if kind == "compute":
                evs.append(TimelineEvent(r + 1, "compute", a, b, label))
            else:
                k = "send_intra" if r // m == peer // m else "send_inter"
                evs.append(TimelineEvent(r + 1, k, a, b, label))
                evs.append(TimelineEvent(peer + 1, "recv", a, b, f"recv {label}"))
    evs.sort(key=lambda e: (e.start, e.device, e.kind, e.label))
    tl = Timeline(evs, max((e.end for e in evs), default=0.0))
    validate_timeline(tl)
    return tl


class ProcessRing:
    """Ring attention for one rank: ``forward`` -> (O, lse); ``backward`` -> (dQ, dK, dV)."""

    def __init__(self, layout: ShardLayout, mask: MaskSpec, topology: Topology | None = None, group=None,
                 head_dim: int | None = None, transport: str | None = None, slots: int | None = None,
                 fanout: int | None = None):
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
        self._trace = None  # list while tracing: (kind, start event, end event, label, peer)
        self._trace_t0 = None
        if transport is None:
            transport = "ce" if self.device.type == "cuda" and self.world > 1 else "collective"
        if slots is None:  # the paper's three buffers per device (fabric.py:87-90): the one being
            slots = min(self.world - 1, 3)  # computed on plus two landing; arena bytes O(1) in G
        if transport not in ("ce", "collective"):
            raise ValueError(f"unknown ring transport {transport!r} (expected 'ce' or 'collective')")
        if transport == "ce" and self.device.type != "cuda":
            raise ValueError("the copy-engine transport needs CUDA devices")
        self.transport = transport
        self.slots = slots  # arena slots per channel (default min(world - 1, 3))
        self.fanout = max(1, int(fanout or os.environ.get("BB_CE_FANOUT", "1")))  # copy streams per push
        self._channels: dict = {}
        self._grad_state: dict = {}  # per gradient channel: partial buffers, their events, fold target
        self.split_own = True  # CE backward: own step split by kv heads around the remote steps
        self._xs_data = self._xs_grad = self._xs_fold = None
        # step s (1..G-1): rank whose shard I hold / rank holding mine
        self._src = [None] + [self.order[t] for t in range(1, self.world)]
        self._dst = [None] + [self._who_had_me(t) for t in range(1, self.world)]

    def _launch(self, fn, *a, label: str = "", **kw):
        if not self.compute:
            return
        if self._trace is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(*a, **kw)
            e1.record()
            self._trace.append(("compute", e0, e1, label or getattr(fn, "__name__", "kernel"), None))
            self.stats.launches += 1
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

    # -------------------------------------------------------------- measured timeline
    def trace_begin(self) -> None:
        """Start recording a measured timeline (CE transport on GPUs): every rank synchronises,
        meets at a barrier and records its time origin, then kernels and pushes are bracketed
        by CUDA events until ``trace_collect``.  Collective."""
        torch.cuda.synchronize(self.device)
        if dist.is_initialized():
            dist.barrier(group=self.group)
        self._trace_t0 = torch.cuda.Event(enable_timing=True)
        self._trace_t0.record()
        self._trace = []

    def trace_collect(self) -> Timeline:
        """Stop recording; gather every rank's events into one validated Timeline in the
        reference's schema (seconds from the barrier).  Collective; every rank gets it."""
        torch.cuda.synchronize(self.device)
        t0 = self._trace_t0
        mine = [(k, t0.elapsed_time(a) / 1e3, t0.elapsed_time(b) / 1e3, lab, peer) for k, a, b, lab, peer in self._trace]
        self._trace = self._trace_t0 = None
        per_rank = [None] * self.world
        if dist.is_initialized() and self.world > 1:
            dist.all_gather_object(per_rank, mine, group=self.group)
        else:
            per_rank = [mine]
        return assemble_timeline(per_rank, self.topology)

    def _push(self, ch, s: int, tensors, stream, lanes, label: str) -> None:
        if self._trace is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ch.push(s, tensors, stream, lanes)
            e1.record(stream)
            self._trace.append(("send", e0, e1, f"{label} {self.rank + 1}->{ch.send_to[s] + 1}", ch.send_to[s]))
        else:
            ch.push(s, tensors, stream, lanes)

    def arena_bytes(self) -> int:
        """Device bytes of this rank's copy-engine arenas (all channels)."""
        return sum(ch.total for ch in self._channels.values())

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
                lse: torch.Tensor | None = None, n_q: int | None = None, o16: torch.Tensor | None = None):
        """Ring forward.  ``n_q`` < n runs only the first n_q query rows (the rows a
        sequence-selective checkpoint dropped, see ``recompute``); K/V still circulate whole.
        ``o16`` (bf16, O's shape): the last launched step also stores bf16(O) there -- the
        operand of the output projection (``layer.project_output_shards``), cast in the
        merge epilogue instead of a separate pass."""
        n, hq, d = q.shape
        if o16 is not None and n_q is not None and n_q < n:
            raise ValueError("o16 is not supported with a partial (n_q < n) forward")
        if n_q is not None and n_q < n:
            o_full = K.fill_(torch.empty(n, hq, d, dtype=torch.float32, device=q.device)) if o is None else o
            lse_full = K.fill_(torch.empty(hq, n, device=q.device), float("-inf")) if lse is None else lse
            saved = self.compute
            self.compute = saved and n_q > 0  # the exchanges are collective: always run them
            try:
                o_p, lse_p = self.forward(q[:n_q].contiguous(), k, v, o_full[:n_q], None)
            finally:
                self.compute = saved
            lse_full[:, :n_q].copy_(lse_p)
            return o_full, lse_full
        o = torch.empty(n, hq, d, dtype=torch.float32, device=q.device) if o is None else o
        lse = torch.empty(hq, n, device=q.device) if lse is None else lse
        # the running state's initialisation (distributed.py:172-173) is compute-lane work that
        # one GPU does too: launched (and traced) like the kernels, skipped with them
        self._launch(K.fill_, o, label="init O")
        self._launch(K.fill_, lse, float("-inf"), label="init lse")
        last = max((t for t in range(self.world) if self.counts[self.rank, self.order[t]]), default=-1)
        if o16 is not None and last < 0 and self.compute:  # nothing visible to this rank: O stays 0
            o16.zero_()
        if self.transport == "ce" and self.world > 1:
            self._forward_ce(q, k, v, o, lse, d, o16, last)
            return o, lse
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
                             self._scale(d), n_q=q.shape[0], o_bf16=o16 if t == last else None)
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
        dq = torch.empty(q.shape, dtype=torch.float32, device=q.device) if dq is None else dq
        dk = torch.empty(k.shape, dtype=torch.float32, device=q.device) if dk is None else dk
        dv = torch.empty(v.shape, dtype=torch.float32, device=q.device) if dv is None else dv
        for t, name in ((dq, "dQ"), (dk, "dK"), (dv, "dV")):
            self._launch(K.fill_, t, label=f"init {name}")
        ce = self.transport == "ce" and self.world > 1
        if kind == BURST_BACKWARD:
            (self._burst_ce if ce else self._burst)(q, k, v, do, lse, delta, dq, dk, dv, d)
        elif kind == RING_BACKWARD:
            (self._ringbwd_ce if ce else self._ringbwd)(q, k, v, do, lse, delta, dq, dk, dv, d)
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
                    K.add_rows_(dq, grad_pending[2])
                    grad_pending = None
                K.fill_(acc)
            if self.counts[j, self.rank]:
                self._launch(K.attn_bwd_step, payload[0], k, v, payload[1], payload[2], payload[3], acc, dk, dv,
                             self.layout, self.dmask, j + 1, self.rank + 1, self._scale(d))
            if t > 0:  # delayed gradient send: my partial for shard j goes to its owner j;
                # I receive the partial for MY shard from the rank that computed it at step t
                if grad_pending is not None:
                    for w in grad_pending[0]:
                        w.wait()
                    K.add_rows_(dq, grad_pending[2])
                box = inbox[t % 2]
                works = self._exchange([acc], [box], j, self._who_had_me(t))
                grad_pending = (works, acc, box)
        if grad_pending is not None:
            for w in grad_pending[0]:
                w.wait()
            K.add_rows_(dq, grad_pending[2])

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
                    K.add_rows_(dk, grad_pending[2][0])
                    K.add_rows_(dv, grad_pending[2][1])
                    grad_pending = None
                K.fill_(acc[0])
                K.fill_(acc[1])
            if self.counts[self.rank, j]:
                self._launch(K.attn_bwd_step, q, kv[0], kv[1], do, lse, delta, dq, acc[0], acc[1],
                             self.layout, self.dmask, self.rank + 1, j + 1, self._scale(d))
            if t > 0:
                if grad_pending is not None:
                    for w in grad_pending[0]:
                        w.wait()
                    K.add_rows_(dk, grad_pending[2][0])
                    K.add_rows_(dv, grad_pending[2][1])
                box = inbox[t % 2]
                works = self._exchange(list(acc), list(box), j, self._who_had_me(t))
                grad_pending = (works, acc, box)
        if grad_pending is not None:
            for w in grad_pending[0]:
                w.wait()
            K.add_rows_(dk, grad_pending[2][0])
            K.add_rows_(dv, grad_pending[2][1])

    # -------------------------------------------------------------- copy-engine transport
    def _channel(self, name: str, tensors, grad: bool):
        """Channel ``name`` for payloads shaped like ``tensors`` (created collectively on first use).
        Data channels carry a shard from its owner to the rank computing on it; gradient
        channels carry the partial computed on a shard back to its owner."""
        spec = [(tuple(t.shape), t.dtype) for t in tensors]
        ch = self._channels.get(name)
        if ch is None or ch.spec != spec:
            from .peer import Channel

            if ch is not None:
                self._quiesce()
                ch.close()
            src, dst = (self._dst, self._src) if grad else (self._src, self._dst)
            ch = Channel(name, spec, src, dst, self.rank, self.world, self.device, self.group, self.slots)
            self._channels[name] = ch
        return ch

    def _streams(self):
        if self._xs_data is None:
            self._xs_data = torch.cuda.Stream(self.device)
            self._xs_grad = torch.cuda.Stream(self.device)
            self._xs_lanes = [[torch.cuda.Stream(self.device) for _ in range(self.fanout - 1)] for _ in range(2)]
            self._xs_fold = torch.cuda.Stream(self.device, priority=-1)  # folds win the next free SM
        return torch.cuda.current_stream(self.device), self._xs_data, self._xs_grad

    def _push_all(self, ch, payload, cs, xs):
        """Queue every step's push of this rank's read-only payload (copy engines, in step order)."""
        ch.begin()
        xs.wait_stream(cs)  # payload produced on the compute stream
        for s in range(1, self.world):
            self._push(ch, s, list(payload), xs, self._xs_lanes[0], f"{ch.name} step {s}")
        self.stats.bytes_sent += (self.world - 1) * ch.payload_bytes

    def _forward_ce(self, q, k, v, o, lse, d, o16=None, last=-1):
        cs, xs, _ = self._streams()
        ch = self._channel("kv", (k, v), grad=False)
        self._push_all(ch, (k, v), cs, xs)
        for t in range(self.world):
            j = self.order[t]
            kv = (k, v) if t == 0 else ch.wait(t, cs)
            if self.counts[self.rank, j]:
                self._launch(K.attn_fwd_step, q, kv[0], kv[1], o, lse, self.layout, self.dmask, self.rank + 1, j + 1,
                             self._scale(d), n_q=q.shape[0], o_bf16=o16 if t == last else None,
                             label=f"forward q{self.rank + 1} x k{j + 1}")
            if t > 0:
                ch.release(t, cs)
        cs.wait_stream(xs)

    def _grad_pass(self, data_name, data, grad_name, own_acc, launch, skip, hkv):
        """Shared copy-engine schedule of both backward passes.

        ``data`` (read-only) is pushed at pass start to every rank that computes on it.  The
        own shard's step is split by kv heads into halves A and B: A runs first, B last.  At
        remote step t the kernel accumulates into a zeroed partial that is pushed to the
        shard's owner as soon as the kernel ends (and re-zeroed on the copy stream behind
        the push).  The owner folds arriving partials into its accumulators on a
        high-priority side stream: everything before B starts, then the last partial's
        A heads while B runs; only the last partial's B heads are added after B."""
        cs, xs, xg = self._streams()
        xf = self._xs_fold
        dch = self._channel(data_name, data, grad=False)
        gch = self._channel(grad_name, own_acc, grad=True)
        self._push_all(dch, data, cs, xs)
        gch.begin()
        st = self._grad_state.get(grad_name)
        if st is None or [tuple(p.shape) for p in st["parts"][0]] != [tuple(a.shape) for a in own_acc]:
            st = {"parts": [tuple(torch.zeros_like(a) for a in own_acc) for _ in range(2)], "free": [None, None]}
            self._grad_state[grad_name] = st
        parts, free = st["parts"], st["free"]  # free[i]: partial buffer i pushed and re-zeroed
        split = self.split_own and hkv >= 2
        hs = [(hkv // 2) * (a.shape[1] // hkv) for a in own_acc]  # first head of half B, per accumulator
        me, last = self.rank, self.world - 1
        if not skip(me):
            self._launch(launch, data, own_acc, me, (0, hkv // 2) if split else None, label=f"{grad_name} own shard A")
        xf.wait_stream(cs)
        b_ready = None
        for t in range(1, self.world):
            j = self.order[t]
            payload = dch.wait(t, cs)
            acc = parts[t % 2]
            if free[t % 2] is not None:
                cs.wait_event(free[t % 2])
            if not skip(j):
                self._launch(launch, payload, acc, j, None, label=f"{grad_name} shard {j + 1} on {me + 1}")
            dch.release(t, cs)
            xg.wait_stream(cs)
            self._push(gch, t, list(acc), xg, self._xs_lanes[1], f"{grad_name} step {t}")
            self.stats.bytes_sent += gch.payload_bytes
            if self.compute:
                with torch.cuda.stream(xg):
                    for x in acc:
                        K.fill_(x)
            ev = torch.cuda.Event()
            ev.record(xg)
            free[t % 2] = ev
            if t == last and split:
                b_ready = torch.cuda.Event()
                b_ready.record(xf)  # every earlier fold (all heads) is done
            views = gch.wait(t, xf)  # the partial of MY shard computed elsewhere at step t
            if self.compute:
                with torch.cuda.stream(xf):
                    for x, g, h in zip(own_acc, views, hs):
                        if t == last and split:
                            K.add_rows_(x[:, :h], g[:, :h])  # half B is being written by the own kernel
                        else:
                            K.add_rows_(x, g)
            if not (t == last and split):
                gch.release(t, xf)
        if split:
            if b_ready is not None:
                cs.wait_event(b_ready)
            if not skip(me):
                self._launch(launch, data, own_acc, me, (hkv // 2, hkv), label=f"{grad_name} own shard B")
            cs.wait_stream(xf)
            if last >= 1:
                views = gch.views(last)
                if self.compute:
                    for x, g, h in zip(own_acc, views, hs):
                        K.add_rows_(x[:, h:], g[:, h:])
                gch.release(last, cs)
        cs.wait_stream(xf)
        cs.wait_stream(xs)
        cs.wait_stream(xg)

    def _burst_ce(self, q, k, v, do, lse, delta, dq, dk, dv, d):
        def launch(payload, acc, j, heads):
            K.attn_bwd_step(payload[0], k, v, payload[1], payload[2], payload[3], acc[0], dk, dv,
                            self.layout, self.dmask, j + 1, self.rank + 1, self._scale(d), kv_heads=heads)

        self._grad_pass("qp", (q, do, lse, delta), "dq", (dq,), launch, lambda j: not self.counts[j, self.rank],
                        k.shape[1])

    def _ringbwd_ce(self, q, k, v, do, lse, delta, dq, dk, dv, d):
        def launch(payload, acc, j, heads):
            K.attn_bwd_step(q, payload[0], payload[1], do, lse, delta, dq, acc[0], acc[1],
                            self.layout, self.dmask, self.rank + 1, j + 1, self._scale(d), kv_heads=heads)

        self._grad_pass("kv", (k, v), "dkv", (dk, dv), launch, lambda j: not self.counts[self.rank, j], k.shape[1])

    def _quiesce(self) -> None:
        """Every rank's earlier passes have finished (so no peer still writes a flag or payload
        into an arena about to be freed): device sync, then a host barrier.  Collective."""
        torch.cuda.synchronize(self.device)
        if dist.is_initialized():
            dist.barrier(group=self.group)

    def close(self) -> None:
        """Release the copy-engine arenas and peer mappings.  Collective (every rank calls it)."""
        if self._channels:
            self._quiesce()
        for ch in self._channels.values():
            ch.close()
        self._channels.clear()
        self._grad_state.clear()

    def _who_had_me(self, t: int) -> int:
        """Rank that computed on MY shard at step t (it sends me that gradient partial)."""
        return next(r for r in range(self.world) if ring_schedule(self.topology, r)[t] == self.rank)


def pass_flops(layout: ShardLayout, mask: MaskSpec, heads: int, head_dim: int) -> tuple[float, float]:
    """Algorithmic FLOPs of the whole job: forward 4*d*H*P, backward 10*d*H*P (FlashAttention
    convention incl. the S recompute; P = exact unmasked pairs)."""
    from .masks import unmasked_pair_count

    p = unmasked_pair_count(mask, layout.seq_len)
    return 4.0 * head_dim * heads * p, 10.0 * head_dim * heads * p
