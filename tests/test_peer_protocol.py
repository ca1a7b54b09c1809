"""Copy-engine ring transport (peer.Channel + ProcessRing "ce" schedule) on a simulated GPU.

Every rank's host code runs for real (ProcessRing forward / burst / ring backward, the
Channel flag protocol), but streams, events and the C-ABI fabric calls are replaced by
a discrete simulation: each stream is a FIFO of operations (kernel, copy, flag write,
flag wait, event record, event wait) that the scheduler executes when their
dependencies are met.  The tests assert that every schedule drains (no deadlock) for
G = 2..8, flat and two-level plans, 1..G-1 arena slots and repeated passes, and that
each push lands in a slot only after its previous reader released it.  This is the CPU
cover for the N > 1 copy-engine path (the GPU runs use 2 and 4 B200s; the driver's
scaling run uses 8).
"""

import ctypes as C
from collections import deque

import pytest
import torch

from paper_2509_19836_b200 import masks as M
from paper_2509_19836_b200 import peer as P
from paper_2509_19836_b200 import ring as R
from paper_2509_19836_b200.fabric import BURST_BACKWARD, RING_BACKWARD, Topology
from paper_2509_19836_b200.partitioning import ShardLayout


class Sim:
    def __init__(self):
        self.mem = {}  # flag address -> value
        self.streams = {}  # handle -> FakeStream
        self.current = {}  # rank -> current stream
        self.rank = 0  # rank whose host code is running
        self.allocs = {}  # rank -> arena count
        self.arenas = {}  # arena base -> Channel
        self.slot_state = {}  # (arena base, slot) -> free / filling / full
        self.violations = []


SIM = None


class Token:
    def __init__(self):
        self.done = False


class FakeStream:
    _next = 1

    def __init__(self, device=None, priority=0):
        self.rank = SIM.rank
        self.q = deque()
        self.cuda_stream = FakeStream._next
        FakeStream._next += 1
        SIM.streams[self.cuda_stream] = self

    def _record(self):
        t = Token()
        self.q.append(("record", t))
        return t

    def wait_stream(self, other):
        self.q.append(("wait", other._record()))

    def wait_event(self, ev):
        if ev.tok is not None:
            self.q.append(("wait", ev.tok))


class FakeEvent:
    def __init__(self, enable_timing=False):
        self.tok = None

    def record(self, stream=None):
        self.tok = (stream or SIM.current[SIM.rank])._record()


class stream_ctx:
    def __init__(self, s):
        self.s = s

    def __enter__(self):
        self.prev = SIM.current[SIM.rank]
        SIM.current[SIM.rank] = self.s

    def __exit__(self, *a):
        SIM.current[SIM.rank] = self.prev


def _val(x):
    return x.value if isinstance(x, C.c_void_p) else int(x)


class FakeLib:
    def bb_ipc_handle_bytes(self):
        return 8

    def bb_arena_alloc(self, total, pref):
        r = SIM.rank
        k = SIM.allocs.get(r, 0)
        SIM.allocs[r] = k + 1
        pref._obj.value = ((r + 1) << 40) | (k << 32)
        return 0

    def bb_ipc_export(self, base, h):
        C.memmove(h, _val(base).to_bytes(8, "little"), 8)
        return 0

    def bb_ipc_import(self, h, qref):
        qref._obj.value = int.from_bytes(bytes(h)[:8], "little")
        return 0

    def bb_copy_async(self, dst, src, nbytes, s):
        SIM.streams[_val(s)].q.append(("copy", _val(dst)))
        return 0

    def bb_flag_write(self, addr, v, s):
        SIM.streams[_val(s)].q.append(("write", _val(addr), int(v)))
        return 0

    def bb_flag_wait(self, addr, v, s):
        SIM.streams[_val(s)].q.append(("flagwait", _val(addr), int(v)))
        return 0

    def bb_ipc_close(self, p):
        return 0

    def bb_arena_free(self, p):
        return 0


class FakeK:
    def device_mask(self, mask, device):
        return None

    def _kernel(self, *reads):
        SIM.current[SIM.rank].q.append(("kernel",))

    def attn_fwd_step(self, *a, **kw):
        self._kernel()

    def attn_bwd_step(self, *a, **kw):
        self._kernel()

    def bwd_preprocess(self, *a, **kw):
        self._kernel()

    def fill_(self, t, value=0.0):
        return t.fill_(value)

    def add_rows_(self, dst, src):
        return dst.add_(src)


def _arena(addr):
    base = addr & ~((1 << 32) - 1)
    return base, SIM.arenas[base]


def _data_slot(addr):
    base, ch = _arena(addr)
    return (base, (addr - base) // ch.slot_bytes)


def _ready_slot(addr):
    base, ch = _arena(addr)
    s = (addr - base - ch.flags_off) // 4
    if addr - base < ch.flags_off or s >= ch.world:
        return None  # a free[] word
    return (base, (s - 1) % ch.slots)


def run_streams():
    progress = True
    while progress:
        progress = False
        for s in SIM.streams.values():
            while s.q:
                op = s.q[0]
                if op[0] == "wait" and not op[1].done:
                    break
                if op[0] == "flagwait" and SIM.mem.get(op[1], 0) < op[2]:
                    break
                s.q.popleft()
                progress = True
                if op[0] == "record":
                    op[1].done = True
                elif op[0] == "write":
                    SIM.mem[op[1]] = op[2]
                    slot = _ready_slot(op[1])
                    if slot is not None:
                        SIM.slot_state[slot] = "full"
                elif op[0] == "copy":
                    slot = _data_slot(op[1])
                    if SIM.slot_state.get(slot) == "full":
                        SIM.violations.append(("overwrite of an unreleased slot", slot))
                    SIM.slot_state[slot] = "filling"
                elif op[0] == "released":
                    SIM.slot_state[op[1]] = "free"
    stuck = [(h, s.rank, list(s.q)[:2]) for h, s in SIM.streams.items() if s.q]
    return stuck


@pytest.fixture
def sim(monkeypatch):
    global SIM
    SIM = Sim()
    FakeStream._next = 1
    monkeypatch.setattr(torch.cuda, "Stream", FakeStream)
    monkeypatch.setattr(torch.cuda, "Event", FakeEvent)
    monkeypatch.setattr(torch.cuda, "stream", stream_ctx)
    monkeypatch.setattr(torch.cuda, "current_stream", lambda device=None: SIM.current[SIM.rank])
    monkeypatch.setattr(P.N, "load", lambda *a, **k: FakeLib())
    monkeypatch.setattr(P, "_arena_tensor", lambda ptr, n, dev: torch.zeros(n, dtype=torch.uint8))
    monkeypatch.setattr(R, "K", FakeK())
    orig_release, orig_init = P.Channel.release, P.Channel.__init__

    def release(self, s, stream):  # mark the slot consumed (in stream order) before handing it on
        stream.q.append(("released", (self.base, self._slot(s))))
        orig_release(self, s, stream)

    def init(self, *a, **k):
        orig_init(self, *a, **k)
        SIM.arenas[self.base] = self

    monkeypatch.setattr(P.Channel, "release", release)
    monkeypatch.setattr(P.Channel, "__init__", init)

    def all_gather_object(out, obj, group=None):
        base = int.from_bytes(obj[:8], "little")
        idx = (base >> 32) & 0xFF
        for r in range(len(out)):
            out[r] = ((((r + 1) << 40) | (idx << 32))).to_bytes(8, "little")

    monkeypatch.setattr(P.dist, "all_gather_object", all_gather_object)
    return SIM


def make_rings(world, topo, slots, hq=2, hkv=2, n_per=8, d=4, fanout=1):
    layout = ShardLayout("zigzag", n_per * world, world)
    rings = []
    for r in range(world):
        SIM.rank = r
        SIM.current[r] = FakeStream()
        ring = R.ProcessRing.__new__(R.ProcessRing)
        # the constructor reads rank / world from torch.distributed: fill the same fields here
        import paper_2509_19836_b200.ring as ring_mod

        orig = (ring_mod.dist.is_initialized, ring_mod.dist.get_world_size, ring_mod.dist.get_rank)
        ring_mod.dist.is_initialized = lambda: True
        ring_mod.dist.get_world_size = lambda g=None: world
        ring_mod.dist.get_rank = lambda g=None, _r=r: _r
        try:
            ring.__init__(layout, M.causal_mask(), Topology(*topo), head_dim=d, transport="collective", slots=slots,
                          fanout=fanout)
        finally:
            ring_mod.dist.is_initialized, ring_mod.dist.get_world_size, ring_mod.dist.get_rank = orig
        ring.transport = "ce"
        rings.append(ring)
    t = lambda h: torch.zeros(n_per, h, d, dtype=torch.bfloat16)  # noqa: E731
    data = [(t(hq), t(hkv), t(hkv), t(hq)) for _ in range(world)]
    return rings, data


def run_pass(rings, data, what):
    """Enqueue one pass on every rank (host code never blocks on the CE path), return state."""
    outs = []
    for r, ring in enumerate(rings):
        SIM.rank = r
        q, k, v, do = data[r]
        if what == "forward":
            outs.append(ring.forward(q, k, v))
        else:
            n, hq, d = q.shape
            o = torch.zeros(n, hq, d)
            lse = torch.zeros(hq, n)
            ring.backward(q, k, v, do, o, lse, kind=what)
    return outs


@pytest.mark.parametrize("world,topo", [(2, (1, 2)), (3, (1, 3)), (4, (1, 4)), (4, (2, 2)), (8, (1, 8)), (8, (2, 4)), (8, (4, 2))])
@pytest.mark.parametrize("slots,fanout", [(None, 1), (1, 1), (2, 1), (None, 3)])
def test_ce_schedule_drains(sim, world, topo, slots, fanout):
    rings, data = make_rings(world, topo, slots, hq=4, hkv=2, fanout=fanout)
    passes = ["forward", BURST_BACKWARD, "forward", RING_BACKWARD, "forward", BURST_BACKWARD, "forward", RING_BACKWARD]
    for i, what in enumerate(passes):
        run_pass(rings, data, what)
        if i % 3 == 2:  # let the GPU run behind the host for a few passes, then drain
            assert run_streams() == []
    assert run_streams() == []
    assert SIM.violations == []
    # every channel saw the same epoch count on every rank
    for name in rings[0]._channels:
        assert len({r._channels[name].epoch for r in rings}) == 1


@pytest.mark.parametrize("world", [2, 4, 8])
def test_ce_schedule_drains_comm_only_and_no_split(sim, world):
    rings, data = make_rings(world, (1, world), None, hq=2, hkv=1)
    for r in rings:
        r.compute = False  # comm-alone timing mode: exchanges without kernels
    for what in ("forward", BURST_BACKWARD, RING_BACKWARD):
        run_pass(rings, data, what)
    assert run_streams() == []
    assert SIM.violations == []


def test_all_passes_enqueued_before_gpu_runs(sim):
    """The host may run many passes ahead of the GPU: flag epochs keep slot reuse safe."""
    rings, data = make_rings(4, (1, 4), 1)
    for _ in range(3):
        for what in ("forward", BURST_BACKWARD):
            run_pass(rings, data, what)
    assert run_streams() == []
    assert SIM.violations == []


def test_simulator_catches_a_missing_release(sim, monkeypatch):
    """Guard on the guard: without the slot hand-over the schedule must deadlock."""
    rings, data = make_rings(4, (1, 4), 1)
    monkeypatch.setattr(P.Channel, "release", lambda self, s, stream: None)
    run_pass(rings, data, "forward")
    assert run_streams() != []
