"""Sequence-level selective checkpointing -- drop-in for burstsim.checkpointing.

Policies and the storage/recompute model are the reference's
(checkpointing.py:36-97).  The difference is that the policy drives the ring
engine: ``checkpoint_states`` keeps (O, lse) only for rows whose global token
id is > round(s*N) (0-based rows [boundary, N), checkpointing.py:141) and frees
the rest; ``recompute_checkpointed`` re-runs the forward ring for exactly the
dropped rows before a backward pass.  Because shard-local token ids increase
with the local row (partitioning.py:96-111), the dropped rows of every device
are a prefix of its shard, so the recompute is the same fwd kernel launched with
n_q = prefix length (with zigzag and s = 0.5 that prefix is the front block).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from .distributed import DeviceState, _plan_for, make_device_states, distributed_forward, burst_backward
from .fabric import Topology
from .masks import MaskSpec, validate_mask
from .partitioning import ShardLayout, pair_count, pair_count_matrix, shard_token_arrays

FULL_RECOMPUTE = "full_recompute"
SELECTIVE_PP = "selective_pp"
SEQUENCE_SELECTIVE = "sequence_selective"
POLICY_KINDS = (FULL_RECOMPUTE, SELECTIVE_PP, SEQUENCE_SELECTIVE)


@dataclass(frozen=True)
class CheckpointPolicy:
    kind: str
    split_fraction: float | None = None

    def __post_init__(self):
        if self.kind not in POLICY_KINDS:
            raise ValueError(f"unknown policy {self.kind!r}, expected {POLICY_KINDS}")
        if self.kind == SEQUENCE_SELECTIVE:
            s = self.split_fraction
            if s is None or not 0.0 < s < 1.0:
                raise ValueError(f"split fraction must lie in (0, 1), got {s}")

    def boundary(self, n: int) -> int:
        """Token index of the split; must land on a whole token (checkpointing.py:48-59)."""
        if self.kind != SEQUENCE_SELECTIVE:
            raise ValueError(f"{self.kind} has no split boundary")
        exact = self.split_fraction * n
        b = round(exact)
        if abs(exact - b) > 1e-9 or not 0 < b < n:
            raise ValueError(f"split fraction {self.split_fraction} does not land on a token boundary for N={n}")
        return int(b)

    def stored_from(self, n: int) -> int:
        """First 0-based row whose (O, lse) is stored."""
        if self.kind == FULL_RECOMPUTE:
            return n
        if self.kind == SELECTIVE_PP:
            return 0
        return self.boundary(n)


@dataclass(frozen=True)
class PlanReport:
    policy: str
    stored_elements_per_layer: int
    recompute_pairs: int
    recompute_fraction: float
    attention_extra_elements: int


def plan(policy: CheckpointPolicy, n: int, d: int, mask: MaskSpec) -> PlanReport:
    """Storage and recompute model (checkpointing.py:71-97); exact pair counts without N x N masks."""
    validate_mask(mask, n)
    ids = np.arange(1, n + 1, dtype=np.int64)
    total = pair_count(mask, ids, ids)
    if policy.kind == FULL_RECOMPUTE:
        stored, rec, extra = n * d, total, 0
    elif policy.kind == SELECTIVE_PP:
        stored, rec, extra = 2 * n * d, 0, n * d
    else:
        b = policy.boundary(n)
        stored, rec, extra = n * d + (n - b) * d, pair_count(mask, ids[:b], ids), (n - b) * d
    return PlanReport(policy.kind, stored, rec, rec / total if total else 0.0, extra)


def _prefix_rows(layout: ShardLayout, stored_from: int) -> list[int]:
    """Per device: number of leading local rows with global id <= stored_from (dropped rows)."""
    return [int(np.searchsorted(ids, stored_from, side="right")) for ids in shard_token_arrays(layout)]


def checkpoint_states(states: list[DeviceState], layout: ShardLayout, policy: CheckpointPolicy) -> list[int]:
    """Keep only the policy's stored (O, lse) rows; returns dropped-prefix length per device."""
    start = policy.stored_from(layout.seq_len)
    prefixes = _prefix_rows(layout, start)
    for st, p in zip(states, prefixes):
        st.o[:p].zero_()  # memory is reused by the recompute; values are gone
        st.lse[:, :p].fill_(float("nan"))
        st.ckpt_prefix = p  # type: ignore[attr-defined]
    return prefixes


def recompute_checkpointed(
    states: list[DeviceState], layout: ShardLayout, mask: MaskSpec, topology: Topology | None = None
) -> int:
    """Recompute the dropped (O, lse) rows with the forward ring restricted to them (K9).
    Returns the number of recomputed query rows summed over devices."""
    plan_ = _plan_for(layout, topology)
    counts = pair_count_matrix(layout, mask)
    total = 0
    for i, st in enumerate(states):
        p = getattr(st, "ckpt_prefix", 0)
        if p == 0:
            continue
        total += p
        hq = st.q.shape[1]
        o_tmp = st.o[:p]  # contiguous row prefix of [n, H, d]
        o_tmp.zero_()
        lse_tmp = torch.full((hq, p), float("-inf"), device=st.device)
        dm = K.device_mask(mask, st.device)
        for t in range(layout.devices):
            j = plan_.visit[i][t]
            if counts[i, j] == 0:
                continue
            src = states[j]
            k_j, v_j = (src.k, src.v) if src.device == st.device else (src.k.to(st.device), src.v.to(st.device))
            with torch.cuda.device(st.device):
                K.attn_fwd_step(st.q[:p], k_j, v_j, o_tmp, lse_tmp, layout, dm, st.index, j + 1, 1.0 / float(np.sqrt(st.head_dim)), n_q=p)
        st.lse[:, :p].copy_(lse_tmp)
        st.ckpt_prefix = 0  # type: ignore[attr-defined]
    return total


@dataclass(frozen=True)
class ToyRunReport:
    policy: str
    recomputed_pairs: int
    stored_elements: int
    max_grad_diff: float
    matches_baseline: bool


def execute_toy(
    policy: CheckpointPolicy, n: int, d: int, mask: MaskSpec, seed: int, tolerance: float = 1e-4, devices=None
) -> ToyRunReport:
    """Run one layer under the policy on the GPU and compare gradients with store-everything
    (checkpointing.py:109-172).  No N <= 64 cap; the tolerance is fp32-level because dQ is
    accumulated with fp32 atomics (order-dependent), everything else is bitwise reproducible."""
    rng = np.random.default_rng(seed)
    q, k, v, do = (rng.uniform(-1.0, 1.0, size=(n, d)) for _ in range(4))
    layout = ShardLayout("contiguous", n, 1)
    base = make_device_states(layout, q, k, v, devices=devices)
    distributed_forward(base, layout, mask)
    burst_backward(base, [do], layout, mask)
    st = make_device_states(layout, q, k, v, devices=devices)
    distributed_forward(st, layout, mask)
    prefixes = checkpoint_states(st, layout, policy)
    recompute_checkpointed(st, layout, mask)
    burst_backward(st, [do], layout, mask)
    diff = max(float((getattr(a, f) - getattr(b, f)).abs().max()) for a, b in zip(st, base) for f in ("dq", "dk", "dv"))
    ids = np.arange(1, n + 1, dtype=np.int64)
    rec_pairs = pair_count(mask, ids[: prefixes[0]], ids) if prefixes[0] else 0
    return ToyRunReport(policy.kind, rec_pairs, plan(policy, n, d, mask).stored_elements_per_layer, diff, diff <= tolerance)
