"""Copy-engine peer channels for the one-process-per-GPU ring (NVLink, no SM work).

The reference moves each ring step's payload with a TransferStep recorded in a
MessageLog (``fabric.py:180-226``; ``distributed.py:176-177, 283-286``).  Here a
:class:`Channel` is one direction of those transfers for one payload kind
(K/V, the burst Q-payload, a gradient partial):

* every rank allocates an *arena* (one ``cudaMalloc``: ``slots`` payload slots +
  32-bit flag words) and exports it by CUDA IPC; peers open it once;
* ``push(s, tensors)`` runs on a copy stream: a copy-engine ``cudaMemcpyAsync``
  of the payload straight into the receiver's slot over NVLink, then a
  ``cuStreamWriteValue32`` of the pass epoch into the receiver's ``ready[s]``;
* ``wait(s)`` makes the consumer stream block on the LOCAL ``ready[s] >= epoch``
  (``cuStreamWaitValue32``) and returns tensor views of the slot;
* ``release(s)`` (after the kernel that read the slot) writes the epoch into
  ``free[s']`` of whichever rank writes that slot next, so a sender never
  overwrites a slot the receiver still reads.

All waits are on local memory and stream-ordered, so nothing blocks the host and
no SM is taken from the attention kernels (NCCL's send/recv are SM kernels that
must wait for an attention CTA to retire before they can run).

Steps are numbered 1..G-1 (step 0 is the rank's own shard, never transferred).
``recv_from[s]`` is the rank whose payload this rank consumes at step ``s`` and
``send_to[s]`` the rank that consumes this rank's payload at step ``s``; each
(step, receiver) pair has exactly one sender, so flag words are single-writer.
"""

from __future__ import annotations

import ctypes as C
import math

import torch
import torch.distributed as dist

from . import _native as N

_ALIGN = 256


def _round_up(x: int, a: int = _ALIGN) -> int:
    return (x + a - 1) // a * a


class _DeviceBytes:
    """__cuda_array_interface__ view of raw device bytes (torch.as_tensor wraps it, no copy)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def _check(rc: int) -> None:
    N.check(rc)


def _arena_tensor(ptr: int, nbytes: int, device: torch.device) -> torch.Tensor:
    """uint8 tensor over an arena's device bytes (no copy, not owned by torch)."""
    return torch.as_tensor(_DeviceBytes(ptr, nbytes), device=device)


class Channel:
    """One payload kind flowing between ring ranks through copy-engine pushes (see module doc)."""

    def __init__(self, name: str, spec: list[tuple[tuple[int, ...], torch.dtype]], recv_from: list[int],
                 send_to: list[int], rank: int, world: int, device: torch.device, group=None, slots: int | None = None):
        self.name = name
        self.spec = [(tuple(s), dt) for s, dt in spec]
        self.rank, self.world, self.device, self.group = rank, world, device, group
        self.recv_from, self.send_to = list(recv_from), list(send_to)  # index 1..world-1 (0 unused)
        steps = world - 1
        self.slots = max(1, min(steps, slots or steps))
        self.sizes = [math.prod(s) * torch.empty((), dtype=dt).element_size() for s, dt in self.spec]
        self.offsets = []
        off = 0
        for b in self.sizes:
            self.offsets.append(off)
            off += _round_up(b)
        self.slot_bytes = _round_up(off)
        self.payload_bytes = sum(self.sizes)
        self.flags_off = self.slots * self.slot_bytes
        total = self.flags_off + _round_up(8 * world)  # ready[world] then free[world], uint32
        lib = N.load()
        p = C.c_void_p()
        _check(lib.bb_arena_alloc(total, C.byref(p)))
        self.base = int(p.value)
        self.total = total
        hbytes = int(lib.bb_ipc_handle_bytes())
        h = (C.c_char * hbytes)()
        _check(lib.bb_ipc_export(C.c_void_p(self.base), h))
        handles: list = [None] * world
        dist.all_gather_object(handles, bytes(h), group=group)
        self.peer_base = [0] * world
        for r in range(world):
            if r == rank:
                self.peer_base[r] = self.base
                continue
            q = C.c_void_p()
            _check(lib.bb_ipc_import(C.create_string_buffer(handles[r], hbytes), C.byref(q)))
            self.peer_base[r] = int(q.value)
        self._lib = lib
        self.arena = _arena_tensor(self.base, total, device)
        self.epoch = 0
        self.bytes_pushed = 0

    # ------------------------------------------------------------ addressing
    def _slot(self, s: int) -> int:
        return (s - 1) % self.slots

    def _ready(self, r: int, s: int) -> int:
        return self.peer_base[r] + self.flags_off + 4 * s

    def _free(self, r: int, s: int) -> int:
        return self.peer_base[r] + self.flags_off + 4 * (self.world + s)

    def views(self, s: int) -> list[torch.Tensor]:
        """Tensor views of this rank's slot for step ``s`` (valid after ``wait(s)``)."""
        base = self._slot(s) * self.slot_bytes
        out = []
        for (shape, dt), off, nb in zip(self.spec, self.offsets, self.sizes):
            out.append(self.arena[base + off: base + off + nb].view(dt).view(shape))
        return out

    # ------------------------------------------------------------ protocol
    def begin(self) -> None:
        """Start a pass (every rank, same order): bumps the epoch the flags carry."""
        self.epoch += 1

    def push(self, s: int, tensors: list[torch.Tensor], stream: torch.cuda.Stream, extra_streams=()) -> None:
        """Copy-engine push of this rank's step-``s`` payload into ``send_to[s]``'s slot.
        ``extra_streams`` split every tensor's bytes across more copy engines; the ready flag
        is written on ``stream`` once all parts have landed."""
        lib, e, dst = self._lib, self.epoch, self.send_to[s]
        h = stream.cuda_stream
        if not (e == 1 and s <= self.slots):  # slot was used before: wait for the receiver's release
            _check(lib.bb_flag_wait(C.c_void_p(self._free(self.rank, s)), e, C.c_void_p(h)))
        lanes = [stream] + list(extra_streams)
        for x in lanes[1:]:
            x.wait_stream(stream)  # payload produced + slot released
        base = self.peer_base[dst] + self._slot(s) * self.slot_bytes
        for t, (shape, dt), off, nb in zip(tensors, self.spec, self.offsets, self.sizes):
            if tuple(t.shape) != shape or t.dtype != dt or not t.is_contiguous():
                raise ValueError(f"channel {self.name}: payload {tuple(t.shape)} {t.dtype} != {shape} {dt}")
            part = _round_up(-(-nb // len(lanes)))
            for i, x in enumerate(lanes):
                lo, hi = i * part, min(nb, (i + 1) * part)
                if hi > lo:
                    _check(lib.bb_copy_async(C.c_void_p(base + off + lo), C.c_void_p(t.data_ptr() + lo), hi - lo,
                                             C.c_void_p(x.cuda_stream)))
        for x in lanes[1:]:
            stream.wait_stream(x)
        _check(lib.bb_flag_write(C.c_void_p(self._ready(dst, s)), e, C.c_void_p(h)))
        self.bytes_pushed += self.payload_bytes

    def wait(self, s: int, stream: torch.cuda.Stream) -> list[torch.Tensor]:
        """Block ``stream`` (not the host) until step ``s``'s payload has landed; return its views."""
        _check(self._lib.bb_flag_wait(C.c_void_p(self._ready(self.rank, s)), self.epoch, C.c_void_p(stream.cuda_stream)))
        return self.views(s)

    def release(self, s: int, stream: torch.cuda.Stream) -> None:
        """After the work on ``stream`` that read slot(s): hand the slot to its next writer."""
        e = self.epoch
        if s + self.slots <= self.world - 1:
            s2, e2 = s + self.slots, e
        else:
            s2, e2 = self._slot(s) + 1, e + 1
        writer = self.recv_from[s2]
        _check(self._lib.bb_flag_write(C.c_void_p(self._free(writer, s2)), e2, C.c_void_p(stream.cuda_stream)))

    def close(self) -> None:
        lib = self._lib
        for r, p in enumerate(self.peer_base):
            if r != self.rank and p:
                lib.bb_ipc_close(C.c_void_p(p))
        self.peer_base = [0] * self.world
        if self.base:
            lib.bb_arena_free(C.c_void_p(self.base))
            self.base = 0
