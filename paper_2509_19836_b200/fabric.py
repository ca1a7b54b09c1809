"""Ring topology, transfer plan and element accounting (fabric.py:45-327 surface).

In burstsim the fabric is a simulator; here it is the *schedule* the engine
executes: ``RingPlan.visit[i][t]`` is the shard device i folds in at ring step
t, and ``transfers`` lists which peer each device's payload goes to.  Inside
one 8xB200 NVSwitch box every hop is a single NVLink traversal, so the 1x8 /
2x4 / 4x2 hierarchies differ in ordering (own shard first vs last, when the
"inter" hop fires) rather than link speed.  ``MessageLog`` keeps the
reference's exact element model; the engine also records the real bytes it
moved.  ``Timeline``/``validate_timeline`` hold *measured* CUDA-event
timelines in the reference's schema (fabric.py:366-388, 674-705).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

DEFAULT_LAT_INTRA = 1e-6
DEFAULT_LAT_INTER = 5e-6
DEFAULT_BW_INTRA = 1e9
DEFAULT_BW_INTER = 1e8

INTRA = "intra"
INTER = "inter"
SCHEDULE_KINDS = ("none", "activation", "gradient")
FORWARD = "forward"
RING_BACKWARD = "ring_backward"
BURST_BACKWARD = "burst_backward"
PASS_KINDS = (FORWARD, RING_BACKWARD, BURST_BACKWARD)


@dataclass(frozen=True)
class Topology:
    num_nodes: int
    gpus_per_node: int
    lat_intra: float = DEFAULT_LAT_INTRA
    lat_inter: float = DEFAULT_LAT_INTER
    bw_intra: float = DEFAULT_BW_INTRA
    bw_inter: float = DEFAULT_BW_INTER

    def __post_init__(self):
        if self.num_nodes < 1 or self.gpus_per_node < 1:
            raise ValueError(
                f"need num_nodes >= 1 and gpus_per_node >= 1, got {self.num_nodes} x {self.gpus_per_node}"
            )
        for name in ("lat_intra", "lat_inter", "bw_intra", "bw_inter"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive, got {getattr(self, name)}")

    @property
    def total_devices(self) -> int:
        return self.num_nodes * self.gpus_per_node

    def link_times(self, payload_elements: float) -> tuple[float, float]:
        return (
            self.lat_intra + payload_elements / self.bw_intra,
            self.lat_inter + payload_elements / self.bw_inter,
        )


def single_node_topology(devices: int) -> Topology:
    return Topology(1, devices)


@dataclass(frozen=True)
class OverlapSchedule:
    kind: str

    def __post_init__(self):
        if self.kind not in SCHEDULE_KINDS:
            raise ValueError(f"unknown schedule {self.kind!r}, expected {SCHEDULE_KINDS}")

    @property
    def buffer_roles(self) -> tuple[str, str, str]:
        return ("compute", "intra_comm", "inter_comm")


def _visit(topology: Topology, dev: int) -> list[int]:
    """0-based shard order for 0-based device ``dev`` (fabric.py:122-139)."""
    r, m = topology.num_nodes, topology.gpus_per_node
    g = r * m
    if g == 1:
        return [0]
    if r == 1:  # flat ring: receive from the predecessor, own shard returns last
        return [(dev - 1 - t) % g for t in range(g)]
    node, slot = divmod(dev, m)  # double ring: own shard first, node-major rounds
    return [((node - a) % r) * m + (slot - b) % m for a in range(r) for b in range(m)]


@dataclass(frozen=True)
class DoubleRing:
    intra_rings: tuple[tuple[int, ...], ...]
    inter_rings: tuple[tuple[int, ...], ...]
    visit_order: tuple[tuple[int, ...], ...]  # 1-based shard ids


def build_double_ring(topology: Topology) -> DoubleRing:
    r, m = topology.num_nodes, topology.gpus_per_node
    intra = tuple(tuple(a * m + b + 1 for b in range(m)) for a in range(r))
    inter = tuple(tuple(a * m + b + 1 for a in range(r)) for b in range(m)) if r > 1 else ()
    visit = tuple(tuple(x + 1 for x in _visit(topology, dev)) for dev in range(topology.total_devices))
    return DoubleRing(intra, inter, visit)


@dataclass(frozen=True)
class TransferStep:
    index: int
    label: str
    channels: tuple[str, ...]
    receiver: tuple[int, ...]


@dataclass(frozen=True)
class RingPlan:
    topology: Topology
    style: str  # single | flat | double
    visit: tuple[tuple[int, ...], ...]
    transfers: tuple[TransferStep, ...]

    @property
    def devices(self) -> int:
        return self.topology.total_devices

    @property
    def steps(self) -> int:
        return self.devices

    def source_of(self, dev: int, step: int) -> int:
        """0-based device that hands ``dev`` its step-``step`` payload (the ring predecessor in the
        plan's order); used by the engine to wire P2P receives."""
        return self.visit[dev][step]


def build_ring_plan(topology: Topology, style: str = "auto") -> RingPlan:
    """fabric.py:166-226: flat = G transfers to dev+1; double = per round m-1 intra + 1 inter."""
    if style not in ("auto", "flat", "double"):
        raise ValueError(f"unknown ring style {style!r}")
    g, r, m = topology.total_devices, topology.num_nodes, topology.gpus_per_node
    if g == 1:
        return RingPlan(topology, "single", ((0,),), ())
    if style == "auto" or (style == "double" and r == 1):
        style = "double" if r > 1 else "flat"
    if style == "flat":
        nxt = tuple((dev + 1) % g for dev in range(g))
        chans = tuple(INTRA if dev // m == nxt[dev] // m else INTER for dev in range(g))
        visit = tuple(tuple((dev - 1 - t) % g for t in range(g)) for dev in range(g))
        steps = tuple(TransferStep(t, f"step {t + 1}", chans, nxt) for t in range(g))
        return RingPlan(topology, "flat", visit, steps)
    intra_rx = tuple((dev // m) * m + (dev % m + 1) % m for dev in range(g))
    inter_rx = tuple(((dev // m + 1) % r) * m + dev % m for dev in range(g))
    steps = []
    for a in range(r):
        for b in range(m - 1):
            steps.append(TransferStep(len(steps), f"round {a + 1} step {b + 1}", (INTRA,) * g, intra_rx))
        steps.append(TransferStep(len(steps), f"round {a + 1} inter", (INTER,) * g, inter_rx))
    visit = tuple(tuple(_visit(topology, dev)) for dev in range(g))
    return RingPlan(topology, "double", visit, tuple(steps))


@dataclass(frozen=True)
class StepRecord:
    index: int
    label: str
    channels: tuple[str, ...]
    receiver: tuple[int, ...]
    elements: int


@dataclass
class MessageLog:
    devices: int
    steps: list[StepRecord] = field(default_factory=list)
    bytes_moved: list[int] = field(default_factory=list)  # real bytes per device (engine-filled)

    def record_plan(self, plan: RingPlan, elements_per_step: int) -> None:
        self.steps.extend(StepRecord(t.index, t.label, t.channels, t.receiver, elements_per_step) for t in plan.transfers)

    def sent(self, device: int, channel: str | None = None) -> int:
        d = device - 1
        return sum(s.elements for s in self.steps if channel is None or s.channels[d] == channel)

    def received(self, device: int, channel: str | None = None) -> int:
        d = device - 1
        return sum(
            s.elements
            for s in self.steps
            for src in range(self.devices)
            if s.receiver[src] == d and (channel is None or s.channels[src] == channel)
        )

    def total_sent(self, device: int) -> int:
        return self.sent(device)

    @property
    def per_device_sent(self) -> tuple[int, ...]:
        return tuple(self.sent(x) for x in range(1, self.devices + 1))

    @property
    def per_device_sent_intra(self) -> tuple[int, ...]:
        return tuple(self.sent(x, INTRA) for x in range(1, self.devices + 1))

    @property
    def per_device_sent_inter(self) -> tuple[int, ...]:
        return tuple(self.sent(x, INTER) for x in range(1, self.devices + 1))

    @property
    def global_sent(self) -> int:
        return sum(self.per_device_sent)

    @property
    def transfer_count(self) -> int:
        return len(self.steps)


def message_log_for(plan: RingPlan, elements_per_step: int) -> MessageLog:
    log = MessageLog(plan.devices)
    log.record_plan(plan, elements_per_step)
    return log


def account_attention_comm(pass_kind: str, seq_len: int, dim: int, devices: int) -> int:
    """Per-device elements per pass: 2Nd / 4Nd / 3Nd + 2N (fabric.py:306-321)."""
    if pass_kind not in PASS_KINDS:
        raise ValueError(f"unknown pass {pass_kind!r}, expected {PASS_KINDS}")
    if devices < 1 or seq_len % devices:
        raise ValueError(f"device count {devices} must divide sequence length {seq_len}")
    return {FORWARD: 2 * seq_len * dim, RING_BACKWARD: 4 * seq_len * dim}.get(pass_kind, 3 * seq_len * dim + 2 * seq_len)


def step_payload_elements(pass_kind: str, seq_len: int, dim: int, devices: int) -> int:
    return account_attention_comm(pass_kind, seq_len, dim, devices) // devices


STRATEGIES = ("ring", "double_ring", "burst")


def analytic_comm_time(strategy: str, topology: Topology, payload_elements: float) -> float:
    """Table-1 closed forms (fabric.py:337-358), kept as the predictor measured timelines are compared to."""
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}, expected {STRATEGIES}")
    t_a, t_e = topology.link_times(payload_elements)
    g, ni = topology.total_devices, topology.num_nodes
    if strategy == "ring":
        return 6.0 * max(g * t_a, g * t_e)
    intra, inter = (g - ni) * t_a, ni * t_e
    if strategy == "double_ring":
        return 4.0 * max(intra, inter) + 2.0 * (intra + inter)
    return 5.0 * max(intra, inter)


@dataclass(frozen=True)
class TimelineEvent:
    device: int  # 1-based
    kind: str  # compute | send_intra | send_inter | recv | buffer_swap
    start: float
    end: float
    label: str


@dataclass
class Timeline:
    events: list[TimelineEvent]
    makespan: float

    def by_kind(self, kind: str) -> list[TimelineEvent]:
        return [e for e in self.events if e.kind == kind]

    def device_events(self, device: int, kind: str | None = None) -> list[TimelineEvent]:
        return [e for e in self.events if e.device == device and (kind is None or e.kind == kind)]


def validate_timeline(timeline: Timeline, tol: float = 1e-12) -> None:
    """Compute lanes never overlap; every recv matches a send; makespan = last end (fabric.py:674-705)."""
    lanes: dict[int, list[TimelineEvent]] = {}
    for e in timeline.events:
        if e.end < e.start:
            raise ValueError(f"event ends before it starts: {e}")
        if e.kind == "compute":
            lanes.setdefault(e.device, []).append(e)
    for dev, evs in lanes.items():
        evs.sort(key=lambda e: e.start)
        for a, b in zip(evs, evs[1:]):
            if b.start < a.end - tol:
                raise ValueError(f"device {dev} compute lane overlaps: {a.label} and {b.label}")
    sends: dict[str, list[TimelineEvent]] = {}
    for e in timeline.events:
        if e.kind.startswith("send_"):
            sends.setdefault(e.label, []).append(e)
    for e in timeline.events:
        if e.kind == "recv":
            cands = sends.get(e.label.removeprefix("recv "), [])
            if not any(math.isclose(s.start, e.start) and math.isclose(s.end, e.end) for s in cands):
                raise ValueError(f"recv without matching send: {e}")
    if timeline.events:
        top = max(e.end for e in timeline.events)
        if not math.isclose(top, timeline.makespan, rel_tol=0, abs_tol=max(tol, 1e-9 * abs(top))):
            raise ValueError(f"makespan {timeline.makespan} != last event end {top}")
