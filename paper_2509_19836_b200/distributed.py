"""BurstAttention ring passes over device shards -- the drop-in for burstsim.distributed.

Same entry points and semantics as the reference (distributed.py:48-351):
``make_device_states`` shards global Q/K/V by a layout, ``distributed_forward``
folds each visiting K/V shard into the running (O, lse) (Alg. 3),
``burst_backward`` keeps K/V resident and circulates (Q, dQ, dO, D, lse)
(Alg. 2), ``ring_backward`` circulates (K, V, dK, dV) (Alg. 1), and
``run_with_schedule`` runs a pass under an overlap schedule.  States are
mutated in place; inputs are never modified; a fresh MessageLog is returned.

What differs is where the work runs.  Each ``DeviceState`` holds bf16 shards
[n, H, d_pad] and fp32 accumulators on a CUDA device (logical device g ->
physical GPU (g-1) mod #GPUs unless ``devices=`` says otherwise), and every
ring step is ONE launch of the sm_100a kernels (bb_attn_fwd_step /
bb_attn_bwd_step) with the visiting payload fetched peer-to-peer on a copy
stream.  2-D inputs ([N, d], the reference's single-head convention) are
treated as one head; results come back in the caller's shape through
``forward_results`` / ``backward_grads`` / ``DeviceState.result``.

This single-process executor is the compatibility path (arbitrary G on any
number of GPUs, visit-order overrides).  The one-process-per-GPU NCCL ring
used for multi-GPU throughput lives in ``ring.py``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import hostio
from . import kernels as K
from .fabric import (
    BURST_BACKWARD,
    FORWARD,
    PASS_KINDS,
    RING_BACKWARD,
    MessageLog,
    OverlapSchedule,
    RingPlan,
    Timeline,
    TimelineEvent,
    Topology,
    build_ring_plan,
    message_log_for,
    single_node_topology,
    step_payload_elements,
    validate_timeline,
)
from .masks import MaskSpec, validate_mask
from .partitioning import ShardLayout, pair_count_matrix, shard_token_arrays


@dataclass(frozen=True)
class AttentionResult:
    o: np.ndarray
    lse: np.ndarray


@dataclass(frozen=True)
class AttentionGrads:
    dq: np.ndarray
    dk: np.ndarray
    dv: np.ndarray


@dataclass
class DeviceState:
    """One device's shards and accumulators (distributed.py:48-60), resident in HBM.

    q: bf16 [n, Hq, d_pad]; k, v: bf16 [n, Hkv, d_pad]; o, dq: fp32 [n, Hq, d_pad];
    lse, d_vec: fp32 [Hq, n]; dk, dv: fp32 [n, Hkv, d_pad].
    """

    index: int  # 1-based
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    o: torch.Tensor | None = None
    lse: torch.Tensor | None = None
    d_vec: torch.Tensor | None = None
    dq: torch.Tensor | None = None
    dk: torch.Tensor | None = None
    dv: torch.Tensor | None = None
    o16: torch.Tensor | None = None  # bf16 copy of O from the last forward step (emit_o_bf16)
    head_dim: int = 0  # unpadded d (softmax scale 1/sqrt(d))
    single_head: bool = False  # caller passed 2-D [N, d] arrays
    token_rows: torch.Tensor | None = field(default=None, repr=False)  # 0-based global rows (int64, device)

    @property
    def device(self) -> torch.device:
        return self.q.device

    def result(self, name: str, out: np.ndarray | None = None) -> np.ndarray:
        """A field as float64 NumPy in the caller's convention ([n, d] for 2-D inputs, lse [n]);
        ``out``: a preallocated float64 array of the field's full shape (``hostio.empty_f64``)."""
        t = getattr(self, name)
        if t is None:
            raise RuntimeError(f"{name} has not been computed")
        a = hostio.to_host_f64(t, out)  # pinned staging + threaded host cast
        if name in ("lse", "d_vec"):
            return a[0] if self.single_head else a
        a = a[..., : self.head_dim]
        return a[:, 0, :] if self.single_head else a


# ----------------------------------------------------------------------------- placement


def _physical_devices(g: int, devices) -> list[torch.device]:
    if devices is not None:
        devs = [torch.device(d) for d in devices]
        if len(devs) != g:
            raise ValueError(f"need {g} devices, got {len(devs)}")
        return devs
    if not torch.cuda.is_available():
        raise RuntimeError("burst-b200 needs CUDA devices (there is no CPU path)")
    n = torch.cuda.device_count()
    return [torch.device("cuda", i % n) for i in range(g)]


def _upload(a: np.ndarray, dev: torch.device) -> torch.Tensor:
    """NumPy [.., d] -> CUDA tensor through pinned staging.  float32 arrays whose d needs no
    padding are cast to the kernels' bf16 on the host (round to nearest even, the same value
    the device cast gives), halving the bytes on PCIe; anything else goes up as float32 and
    is cast (and padded) on the device, as before."""
    if a.dtype == np.float32 and a.shape[-1] == K.padded_head_dim(a.shape[-1]):
        return hostio.to_device(a, dev, torch.bfloat16)
    return hostio.to_device(a, dev)


def _as_global(x, name: str, dev: torch.device) -> tuple[torch.Tensor, bool]:
    """Caller array -> CUDA tensor [N, H, d] (fp32 or bf16), plus 'was 2-D'."""
    if isinstance(x, np.ndarray) or not isinstance(x, torch.Tensor):
        a = np.asarray(x)
        two_d = a.ndim == 2
        if two_d:
            a = a[:, None, :]
        if a.ndim != 3:
            raise ValueError(f"{name} must be [N, d] or [N, H, d], got shape {tuple(a.shape)}")
        return _upload(a, dev), two_d  # via pinned staging
    t = x
    two_d = t.ndim == 2
    if two_d:
        t = t[:, None, :]
    if t.ndim != 3:
        raise ValueError(f"{name} must be [N, d] or [N, H, d], got shape {tuple(t.shape)}")
    if t.dtype not in (torch.bfloat16, torch.float32):
        t = t.to(torch.float32)
    return t.to(dev), two_d


def _to_kernel_bf16(t: torch.Tensor, d_pad: int) -> torch.Tensor:
    if t.dtype == torch.bfloat16 and t.shape[-1] == d_pad:
        return t.contiguous()
    return K.cast_pad_bf16(t.float().contiguous(), d_pad)


def _shard(t: torch.Tensor, rows: torch.Tensor, dev: torch.device) -> torch.Tensor:
    """Row gather through the permute kernel (K5), then placement on ``dev``."""
    out = torch.empty((rows.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    K.permute_rows(out, t, rows.to(t.device), scatter=False)
    return out if out.device == dev else out.to(dev)


def make_device_states(layout: ShardLayout, q, k, v, devices=None) -> list[DeviceState]:
    """Shard global Q/K/V ([N, d] or [N, H, d]) into per-device states (distributed.py:104-115)."""
    devs = _physical_devices(layout.devices, devices)
    qg, two_d = _as_global(q, "Q", devs[0])
    kg, _ = _as_global(k, "K", devs[0])
    vg, _ = _as_global(v, "V", devs[0])
    if qg.shape[0] != layout.seq_len:
        raise ValueError(f"Q has {qg.shape[0]} rows, layout expects {layout.seq_len}")
    if kg.shape != vg.shape or kg.shape[0] != qg.shape[0] or kg.shape[2] != qg.shape[2]:
        raise ValueError("Q, K, V must share N and the head dimension, and K/V must match")
    if qg.shape[1] % kg.shape[1]:
        raise ValueError(f"query heads {qg.shape[1]} must be a multiple of key/value heads {kg.shape[1]}")
    d = int(qg.shape[2])
    d_pad = K.padded_head_dim(d)
    qb, kb, vb = (_to_kernel_bf16(t, d_pad) for t in (qg, kg, vg))
    states = []
    for i, ids in enumerate(shard_token_arrays(layout)):
        rows = torch.from_numpy(ids - 1).to(devs[0])
        st = DeviceState(
            index=i + 1,
            q=_shard(qb, rows, devs[i]),
            k=_shard(kb, rows, devs[i]),
            v=_shard(vb, rows, devs[i]),
            head_dim=d,
            single_head=two_d,
            token_rows=rows.to(devs[i]),
        )
        states.append(st)
    return states


def shard_rows(layout: ShardLayout, x) -> list:
    """Per-device row blocks of a global array (distributed.py:118-119); NumPy in -> NumPy out."""
    ids = shard_token_arrays(layout)
    if isinstance(x, torch.Tensor):
        out = []
        for r in ids:
            rows = torch.from_numpy(r - 1).to(x.device)
            o = torch.empty((len(r),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
            if x.is_cuda and x.is_contiguous() and (x[0].numel() * x.element_size()) % 16 == 0:
                K.permute_rows(o, x, rows, scatter=False)
            else:
                o = x[rows]
            out.append(o)
        return out
    x = np.asarray(x)
    return [_take_rows(x, r - 1) for r in ids]


def _take_rows(x: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """x[rows] (a new array, like the reference's fancy index) for the sorted runs every
    layout's shard is made of: one block copy per run on torch's thread pool instead of
    NumPy's single-threaded per-row gather."""
    breaks = np.flatnonzero(np.diff(rows) != 1) + 1
    if len(rows) == 0 or len(breaks) > 64 or not x.flags.c_contiguous or x.dtype.kind not in "fiub":
        return x[rows]
    starts = np.concatenate([[0], breaks]).astype(np.int64)
    ends = np.concatenate([breaks, [len(rows)]]).astype(np.int64)
    out = np.empty((len(rows),) + x.shape[1:], dtype=x.dtype)
    for a, b in zip(starts, ends):
        r0 = int(rows[a])
        torch.from_numpy(out[a:b]).copy_(torch.from_numpy(x[r0: r0 + (b - a)]))
    return out


def gather_rows(layout: ShardLayout, shard_arrays: list):
    """Reassemble per-shard rows into global token order (distributed.py:122-130)."""
    ids = shard_token_arrays(layout)
    first = shard_arrays[0]
    if isinstance(first, torch.Tensor):
        dev = first.device
        out = torch.zeros((layout.seq_len,) + tuple(first.shape[1:]), dtype=first.dtype, device=dev)
        for r, a in zip(ids, shard_arrays):
            a = a.to(dev).contiguous()
            rows = torch.from_numpy(r - 1).to(dev)
            if dev.type == "cuda" and (a[0].numel() * a.element_size()) % 16 == 0:
                K.permute_rows(out, a, rows, scatter=True)
            else:
                out[rows] = a
        return out
    out = np.zeros((layout.seq_len,) + np.asarray(first).shape[1:], dtype=np.float64)
    for r, a in zip(ids, shard_arrays):
        out[r - 1] = a
    return out


# ----------------------------------------------------------------------------- ring execution


def _plan_for(layout: ShardLayout, topology: Topology | None) -> RingPlan:
    topo = topology if topology is not None else single_node_topology(layout.devices)
    if topo.total_devices != layout.devices:
        raise ValueError(f"topology has {topo.total_devices} devices but layout shards {layout.devices}")
    return build_ring_plan(topo)


class _Executor:
    """Streams, events and payload fetches for one pass over G logical devices."""

    def __init__(self, states: list[DeviceState], overlap: bool, record: bool):
        self.states = states
        self.overlap = overlap
        self.record = record
        self.copy_streams: dict[torch.device, torch.cuda.Stream] = {}
        self.events: list[tuple] = []  # (device, kind, start_evt, end_evt, label)
        self.bytes = [0] * len(states)
        self.t0 = {}
        for st in states:
            if st.device not in self.t0:
                e = torch.cuda.Event(enable_timing=True)
                e.record(torch.cuda.current_stream(st.device))
                self.t0[st.device] = e

    def fetch(self, tensors: tuple[torch.Tensor, ...], dst: torch.device, src_index: int, dst_index: int, label: str):
        """Bring a payload to ``dst`` (peer copy on a copy stream when the owner lives elsewhere)."""
        if all(t.device == dst for t in tensors):
            return tensors
        cs = self.copy_streams.get(dst)
        if cs is None:
            cs = torch.cuda.Stream(dst) if self.overlap else torch.cuda.current_stream(dst)
            self.copy_streams[dst] = cs
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(dst):
            for t in tensors:  # the source stream's writes must be complete before the copy
                cs.wait_event(self._src_ready(t.device))
            start.record(cs)
            with torch.cuda.stream(cs):
                out = tuple(t.to(dst, non_blocking=True) for t in tensors)
            end.record(cs)
            torch.cuda.current_stream(dst).wait_event(end)
            for t in out:  # allocated on the copy stream, consumed on the compute stream
                t.record_stream(torch.cuda.current_stream(dst))
        nbytes = sum(t.numel() * t.element_size() for t in tensors)
        self.bytes[src_index] += nbytes
        if self.record:
            self.events.append((dst_index, "recv", start, end, label, src_index))
        return out

    def _src_ready(self, dev: torch.device) -> torch.cuda.Event:
        e = torch.cuda.Event()
        e.record(torch.cuda.current_stream(dev))
        return e

    def compute(self, dev_index: int, label: str, fn):
        st = self.states[dev_index]
        with torch.cuda.device(st.device):
            s = torch.cuda.current_stream(st.device)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
        if self.record:
            self.events.append((dev_index, "compute", a, b, label, None))

    def timeline(self) -> Timeline:
        for dev in self.t0:
            torch.cuda.synchronize(dev)
        evs = []
        for dev_index, kind, a, b, label, src in self.events:
            base = self.t0[self.states[dev_index].device]
            s, e = base.elapsed_time(a) / 1e3, base.elapsed_time(b) / 1e3
            if kind == "recv":
                evs.append(TimelineEvent(src + 1, "send_intra", s, e, label))
                evs.append(TimelineEvent(dev_index + 1, "recv", s, e, f"recv {label}"))
            else:
                evs.append(TimelineEvent(dev_index + 1, kind, s, e, label))
        evs.sort(key=lambda x: (x.start, x.device, x.kind, x.label))
        return Timeline(evs, max((x.end for x in evs), default=0.0))


def _scale(st: DeviceState) -> float:
    return 1.0 / float(np.sqrt(st.head_dim))


def _check_states(states: list[DeviceState], layout: ShardLayout) -> None:
    if len(states) != layout.devices:
        raise ValueError(f"{len(states)} states for a layout of {layout.devices} devices")


def distributed_forward(
    states: list[DeviceState],
    layout: ShardLayout,
    mask: MaskSpec,
    topology: Topology | None = None,
    visit_order: list[list[int]] | None = None,
    schedule: OverlapSchedule | None = None,
    _exec: _Executor | None = None,
    emit_o_bf16: bool = False,
) -> MessageLog:
    """Ring forward (Alg. 3): fills each state's (o, lse) in place (distributed.py:151-195).

    ``emit_o_bf16``: each device's last launched step also stores bf16(O) into ``state.o16``
    (the cast the output projection's GEMM needs, fused into the merge epilogue)."""
    _check_states(states, layout)
    validate_mask(mask, layout.seq_len)
    plan = _plan_for(layout, topology)
    order = visit_order if visit_order is not None else plan.visit
    counts = pair_count_matrix(layout, mask)
    g = layout.devices
    ex = _exec or _Executor(states, overlap=(schedule is None or schedule.kind != "none"), record=False)
    for st in states:
        st.o = K.fill_(torch.empty(st.q.shape, dtype=torch.float32, device=st.device))
        st.lse = K.fill_(torch.empty(st.q.shape[1], st.q.shape[0], device=st.device), float("-inf"))
    masks = {st.device: K.device_mask(mask, st.device) for st in states}
    last = [max((t for t in range(g) if counts[i, order[i][t]]), default=-1) for i in range(g)]
    for i, st in enumerate(states):
        st.o16 = torch.empty(st.q.shape, dtype=torch.bfloat16, device=st.device) if emit_o_bf16 else None
    for t in range(g):
        for i, st in enumerate(states):
            j = order[i][t]
            if counts[i, j] == 0:
                continue  # compute skipped; the ring step itself is still accounted (:178-179)
            src = states[j]
            k_j, v_j = ex.fetch((src.k, src.v), st.device, j, i, f"fwd step {t + 1} kv {j + 1}->{i + 1}")
            o16 = st.o16 if t == last[i] else None
            ex.compute(
                i,
                f"fwd step {t + 1} shard {j + 1}",
                lambda st=st, k_j=k_j, v_j=v_j, j=j, o16=o16: K.attn_fwd_step(
                    st.q, k_j, v_j, st.o, st.lse, layout, masks[st.device], st.index, j + 1, _scale(st), o_bf16=o16
                ),
            )
    for st in states:  # a globally fully-masked row is an error (distributed.py:189-194)
        bad = torch.isneginf(st.lse)
        if bool(bad.any()):
            row = int(bad.any(dim=0).nonzero()[0, 0]) + 1
            raise ValueError(f"device {st.index} query row {row} has no unmasked key globally")
    log = message_log_for(plan, step_payload_elements(FORWARD, layout.seq_len, states[0].head_dim, g))
    log.bytes_moved = list(ex.bytes)
    return log


def forward_results(states: list[DeviceState]) -> list[AttentionResult]:
    return [AttentionResult(o=st.result("o"), lse=st.result("lse")) for st in states]


def _require_forward(states: list[DeviceState], what: str) -> None:
    if any(st.o is None or st.lse is None for st in states):
        raise RuntimeError(f"{what} requires a completed forward pass (O, Lse missing)")


def _do_shards(states: list[DeviceState], do_shards) -> list[torch.Tensor]:
    out = []
    for st, d in zip(states, do_shards):
        host = not isinstance(d, torch.Tensor)
        t = np.asarray(d) if host else d
        if t.ndim == 2:
            t = t[:, None, :]
        if t.shape[0] != st.q.shape[0] or t.shape[1] != st.q.shape[1]:
            raise ValueError(f"dO shard for device {st.index} has shape {tuple(t.shape)}, expected {tuple(st.q.shape[:2])} x d")
        if host:
            t = _upload(t, st.device)
        elif t.dtype not in (torch.bfloat16, torch.float32):
            t = t.to(torch.float32)
        out.append(_to_kernel_bf16(t.to(st.device), st.q.shape[2]))
    return out


def burst_backward(
    states: list[DeviceState],
    do_shards,
    layout: ShardLayout,
    mask: MaskSpec,
    topology: Topology | None = None,
    schedule: OverlapSchedule | None = None,
    _exec: _Executor | None = None,
) -> MessageLog:
    """Alg. 2 (distributed.py:255-299): K/V resident; (Q_j, dQ_j, dO_j, D_j, Lse_j) circulate.

    D_j = rowsum(dO_j o O_j) is computed once (bb_attn_bwd_preprocess).  The
    device holding payload j accumulates its dQ_j contribution into a local fp32
    partial that is added into the circulating dQ_j (the delayed-gradient send
    of PAPER.md:354); with a single GPU the partial is dQ_j itself."""
    _require_forward(states, "burst_backward")
    _check_states(states, layout)
    validate_mask(mask, layout.seq_len)
    plan = _plan_for(layout, topology)
    counts = pair_count_matrix(layout, mask)
    g = layout.devices
    dos = _do_shards(states, do_shards)
    ex = _exec or _Executor(states, overlap=(schedule is None or schedule.kind != "none"), record=False)
    masks = {st.device: K.device_mask(mask, st.device) for st in states}
    for st, do_i in zip(states, dos):
        st.d_vec = torch.empty_like(st.lse)
        with torch.cuda.device(st.device):
            K.bwd_preprocess(do_i, st.o, st.d_vec)
        st.dk = K.fill_(torch.empty(st.k.shape, dtype=torch.float32, device=st.device))
        st.dv = K.fill_(torch.empty(st.v.shape, dtype=torch.float32, device=st.device))
        st.dq = K.fill_(torch.empty(st.q.shape, dtype=torch.float32, device=st.device))
    for t in range(g):
        for i, st in enumerate(states):
            j = plan.visit[i][t]
            if counts[j, i] == 0:
                continue
            src = states[j]
            q_j, do_j, lse_j, d_j = ex.fetch((src.q, dos[j], src.lse, src.d_vec), st.device, j, i, f"bwd step {t + 1} q {j + 1}->{i + 1}")
            local = src.dq.device == st.device
            dq_acc = src.dq if local else K.fill_(torch.empty(src.q.shape, dtype=torch.float32, device=st.device))
            ex.compute(
                i,
                f"bwd step {t + 1} shard {j + 1}",
                lambda st=st, q_j=q_j, do_j=do_j, lse_j=lse_j, d_j=d_j, dq_acc=dq_acc, j=j: K.attn_bwd_step(
                    q_j, st.k, st.v, do_j, lse_j, d_j, dq_acc, st.dk, st.dv, layout, masks[st.device], j + 1, st.index, _scale(st)
                ),
            )
            if not local:
                (back,) = ex.fetch((dq_acc,), src.device, i, j, f"bwd step {t + 1} dq {i + 1}->{j + 1}")
                with torch.cuda.device(src.device):
                    K.add_rows_(src.dq, back)
    log = message_log_for(plan, step_payload_elements(BURST_BACKWARD, layout.seq_len, states[0].head_dim, g))
    log.bytes_moved = list(ex.bytes)
    return log


def ring_backward(
    states: list[DeviceState],
    do_shards,
    layout: ShardLayout,
    mask: MaskSpec,
    topology: Topology | None = None,
    schedule: OverlapSchedule | None = None,
    _exec: _Executor | None = None,
) -> MessageLog:
    """Alg. 1 (distributed.py:207-252): K, V, dK, dV circulate; dQ stays local."""
    _require_forward(states, "ring_backward")
    _check_states(states, layout)
    validate_mask(mask, layout.seq_len)
    plan = _plan_for(layout, topology)
    counts = pair_count_matrix(layout, mask)
    g = layout.devices
    dos = _do_shards(states, do_shards)
    ex = _exec or _Executor(states, overlap=(schedule is None or schedule.kind != "none"), record=False)
    masks = {st.device: K.device_mask(mask, st.device) for st in states}
    for st, do_i in zip(states, dos):
        st.d_vec = torch.empty_like(st.lse)
        with torch.cuda.device(st.device):
            K.bwd_preprocess(do_i, st.o, st.d_vec)
        st.dq = K.fill_(torch.empty(st.q.shape, dtype=torch.float32, device=st.device))
        st.dk = K.fill_(torch.empty(st.k.shape, dtype=torch.float32, device=st.device))
        st.dv = K.fill_(torch.empty(st.v.shape, dtype=torch.float32, device=st.device))
    for t in range(g):
        for i, st in enumerate(states):
            j = plan.visit[i][t]
            if counts[i, j] == 0:
                continue
            src = states[j]
            k_j, v_j = ex.fetch((src.k, src.v), st.device, j, i, f"rbwd step {t + 1} kv {j + 1}->{i + 1}")
            local = src.dk.device == st.device
            dk_acc = src.dk if local else K.fill_(torch.empty(src.k.shape, dtype=torch.float32, device=st.device))
            dv_acc = src.dv if local else K.fill_(torch.empty(src.v.shape, dtype=torch.float32, device=st.device))
            ex.compute(
                i,
                f"rbwd step {t + 1} shard {j + 1}",
                lambda st=st, k_j=k_j, v_j=v_j, dk_acc=dk_acc, dv_acc=dv_acc, i=i, j=j: K.attn_bwd_step(
                    st.q, k_j, v_j, dos[i], st.lse, st.d_vec, st.dq, dk_acc, dv_acc, layout, masks[st.device], st.index, j + 1, _scale(st)
                ),
            )
            if not local:
                back_k, back_v = ex.fetch((dk_acc, dv_acc), src.device, i, j, f"rbwd step {t + 1} dkv {i + 1}->{j + 1}")
                with torch.cuda.device(src.device):
                    K.add_rows_(src.dk, back_k)
                    K.add_rows_(src.dv, back_v)
    log = message_log_for(plan, step_payload_elements(RING_BACKWARD, layout.seq_len, states[0].head_dim, g))
    log.bytes_moved = list(ex.bytes)
    return log


def backward_grads(states: list[DeviceState]) -> list[AttentionGrads]:
    # The backward kernels are still running when a caller gets here (nothing in the passes
    # waits for them): allocate and page in every float64 result first, so that host work
    # overlaps the GPU and the copies afterwards write to resident pages.
    names = ("dq", "dk", "dv")
    for st in states:
        for name in names:
            if getattr(st, name) is None:
                raise RuntimeError(f"{name} has not been computed")
    outs = [{name: hostio.empty_f64(getattr(st, name)) for name in names} for st in states]
    return [AttentionGrads(**{name: st.result(name, o[name]) for name in names}) for st, o in zip(states, outs)]


@dataclass
class ScheduledRun:
    results: list
    message_log: MessageLog
    timeline: Timeline


def run_with_schedule(
    pass_kind: str,
    layout: ShardLayout,
    mask: MaskSpec,
    q,
    k,
    v,
    do=None,
    topology: Topology | None = None,
    schedule: OverlapSchedule | None = None,
    compute_time_per_step: float = 1e-3,
    devices=None,
) -> ScheduledRun:
    """Run a pass under a schedule (distributed.py:313-351).  Values do not depend on the
    schedule; the timeline is MEASURED (CUDA events per ring step and per peer copy, in the
    reference's Timeline schema) instead of simulated, so ``compute_time_per_step`` is unused."""
    if pass_kind not in PASS_KINDS:
        raise ValueError(f"unknown pass {pass_kind!r}, expected {PASS_KINDS}")
    topo = topology if topology is not None else single_node_topology(layout.devices)
    schedule = schedule if schedule is not None else OverlapSchedule("none")
    if pass_kind != FORWARD and do is None:
        raise ValueError("backward passes need the output cotangent dO")
    states = make_device_states(layout, q, k, v, devices=devices)
    ex = _Executor(states, overlap=schedule.kind != "none", record=True)
    log = distributed_forward(states, layout, mask, topo, schedule=schedule, _exec=ex)
    if pass_kind == FORWARD:
        results: list = forward_results(states)
    else:
        do_shards = shard_rows(layout, do if isinstance(do, torch.Tensor) else np.asarray(do, dtype=np.float64))
        fn = ring_backward if pass_kind == RING_BACKWARD else burst_backward
        log = fn(states, do_shards, layout, mask, topo, schedule=schedule, _exec=ex)
        results = backward_grads(states)
    timeline = ex.timeline()
    validate_timeline(timeline)
    return ScheduledRun(results=results, message_log=log, timeline=timeline)
