"""BurstAttention as a differentiable torch op on one rank's sequence shard.

The reference is a simulator with explicit forward / backward calls
(``distributed_forward`` then ``burst_backward`` / ``ring_backward``,
distributed.py:151-299); a training stack (the paper's BMTrain/FSDP integration,
PAPER.md:584) needs the same ring as an autograd node.  ``BurstAttention.apply``
runs :meth:`ProcessRing.forward` and saves what the chosen backward needs; its
backward runs the ring backward pass with the incoming dO.  With a
``sequence_selective`` :class:`~.checkpointing.CheckpointPolicy` only the kept
suffix of (O, lse) is saved and the dropped prefix is recomputed by the ring
before the backward pass (checkpointing.py:141-157), so the saved activation
shrinks by the policy's fraction.
"""

from __future__ import annotations

import torch

from .checkpointing import SEQUENCE_SELECTIVE, CheckpointPolicy, _prefix_rows
from .fabric import BURST_BACKWARD


class BurstAttention(torch.autograd.Function):
    """``(O, lse) = BurstAttention.apply(q, k, v, ring, backward_kind, policy)`` on this rank's shard."""

    @staticmethod
    def forward(ctx, q, k, v, ring, backward_kind=BURST_BACKWARD, policy: CheckpointPolicy | None = None):
        o, lse = ring.forward(q, k, v)
        drop = 0
        if policy is not None and policy.kind == SEQUENCE_SELECTIVE:
            drop = _prefix_rows(ring.layout, policy.stored_from(ring.layout.seq_len))[ring.rank]
        ctx.ring, ctx.kind, ctx.policy, ctx.drop = ring, backward_kind, policy, drop
        if drop:
            ctx.save_for_backward(q, k, v, o[drop:].clone(), lse[:, drop:].clone())
        else:
            ctx.save_for_backward(q, k, v, o, lse)
        ctx.mark_non_differentiable(lse)
        return o, lse

    @staticmethod
    def backward(ctx, do, _dlse):
        q, k, v, o_kept, lse_kept = ctx.saved_tensors
        ring, drop = ctx.ring, ctx.drop
        if drop:  # rebuild the dropped prefix (a collective: every rank takes part)
            n, hq, d = q.shape
            o = torch.empty(n, hq, d, dtype=o_kept.dtype, device=o_kept.device)
            lse = torch.empty(hq, n, dtype=lse_kept.dtype, device=lse_kept.device)
            o[drop:] = o_kept
            lse[:, drop:] = lse_kept
            ring.recompute(q, k, v, o, lse, ctx.policy)
        else:
            o, lse = o_kept, lse_kept
            if ctx.policy is not None and ctx.policy.kind == SEQUENCE_SELECTIVE:
                ring.recompute(q, k, v, o, lse, ctx.policy)  # nothing dropped here: exchanges only
        do = do.to(q.dtype).contiguous()
        dq, dk, dv = ring.backward(q, k, v, do, o, lse, kind=ctx.kind)
        return dq.to(q.dtype), dk.to(k.dtype), dv.to(v.dtype), None, None, None


def burst_attention(q, k, v, ring, backward_kind: str = BURST_BACKWARD, policy: CheckpointPolicy | None = None):
    """Differentiable ring attention output O (float32, [n, Hq, d]) for this rank's shard."""
    o, _ = BurstAttention.apply(q, k, v, ring, backward_kind, policy)
    return o
