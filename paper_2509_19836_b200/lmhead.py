"""Fused LM head + cross entropy -- drop-in for burstsim.lmhead (lmhead.py:21-116).

``fused_lmhead_loss(h, w_head, targets, cfg)`` returns per-token losses (the
caller sums, oracle.py:129-133), dH and dW with the reference's sign
convention (softmax - onehot) and ``peak_aux_elements`` =
min(B_s, N) * V, the one retained logits row tile (lmhead.py:73-74).

On the B200 each row tile is: a tcgen05 GEMM H.W^T whose epilogue writes the
fp32 logits tile plus per-(row, 256-vocab tile) (max, sum exp) partials and the
target logit; an LSE combine; an in-place softmax - onehot to bf16; and two
tcgen05 GEMMs for dH (= G.W) and dW (+= G^T.H) that read G and W / H through
MN-major descriptors (no transposes).  Logits are never recomputed (6NVD
FLOPs).  dW accumulates in fp32 across row tiles and, under
torch.distributed, across sequence shards (``all_reduce_dw``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K


@dataclass(frozen=True)
class FusionConfig:
    rows_per_tile: int  # B_s
    vocab_per_tile: int  # B_v

    def __post_init__(self):
        if self.rows_per_tile < 1 or self.vocab_per_tile < 1:
            raise ValueError(
                f"tile sizes must be >= 1, got rows={self.rows_per_tile}, vocab={self.vocab_per_tile}"
            )


@dataclass
class FusedLossResult:
    loss: object  # per-token nats: np.ndarray (NumPy callers) or fp32 tensor
    dh: object
    dw: object
    peak_aux_elements: int


def _pad_cols(x: torch.Tensor, cols: int) -> torch.Tensor:
    if x.dtype == torch.bfloat16 and x.shape[1] == cols and x.is_contiguous():
        return x
    return K.cast_pad_bf16(x.float().contiguous(), cols)


def fused_lmhead_loss(h, w_head, targets, cfg: FusionConfig, device=None, dw_out: torch.Tensor | None = None) -> FusedLossResult:
    """Fused forward + backward (lmhead.py:41-93) on one GPU.

    NumPy inputs give NumPy float64 outputs in the reference's shapes; torch
    inputs give fp32 CUDA tensors.  ``dw_out`` (fp32 [V, D_pad]) accumulates dW
    in place, e.g. across sequence shards before an all-reduce."""
    numpy_io = not isinstance(h, torch.Tensor)
    dev = torch.device(device) if device is not None else (h.device if not numpy_io and h.is_cuda else torch.device("cuda", torch.cuda.current_device()))
    ht = torch.as_tensor(h).to(dev)
    wt = torch.as_tensor(w_head).to(dev)
    y = torch.as_tensor(np.asarray(targets, dtype=np.int64) if not isinstance(targets, torch.Tensor) else targets).to(dev, torch.int64)
    if ht.ndim != 2 or wt.ndim != 2:
        raise ValueError("H and W_head must be 2-dimensional")
    n, d = ht.shape
    v = wt.shape[0]
    if wt.shape[1] != d:
        raise ValueError(f"W_head must have {d} columns, got {wt.shape[1]}")
    if tuple(y.shape) != (n,):
        raise ValueError(f"targets must have length {n}, got shape {tuple(y.shape)}")
    bad = (y < 0) | (y >= v)
    if bool(bad.any()):
        r = int(bad.nonzero()[0, 0])
        raise ValueError(f"target index {int(y[r])} at row {r} outside [0, {v})")
    d_pad = max(8, (d + 7) // 8 * 8)
    hb = _pad_cols(ht, d_pad)
    wb = _pad_cols(wt, d_pad)
    loss = torch.empty(n, dtype=torch.float32, device=dev)
    dh = torch.empty(n, d_pad, dtype=torch.float32, device=dev)
    dw = dw_out if dw_out is not None else torch.zeros(v, d_pad, dtype=torch.float32, device=dev)
    rows = min(cfg.rows_per_tile, n)
    ws = torch.empty(K.lmhead_workspace_bytes(n, v, d_pad, rows), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        K.lmhead_fused(hb, wb, y.contiguous(), loss, dh, dw, rows, cfg.vocab_per_tile, ws)
    peak = rows * v
    if numpy_io:
        return FusedLossResult(
            loss=loss.double().cpu().numpy(),
            dh=dh[:, :d].double().cpu().numpy(),
            dw=dw[:, :d].double().cpu().numpy(),
            peak_aux_elements=peak,
        )
    return FusedLossResult(loss=loss, dh=dh[:, :d], dw=dw[:, :d] if dw_out is None else dw, peak_aux_elements=peak)


def all_reduce_dw(dw: torch.Tensor, group=None) -> torch.Tensor:
    """K8: sum dW over sequence shards (one NCCL all-reduce at the end of the LM-head backward)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(dw, group=group)
    return dw


@dataclass
class ShardedLossResult:
    """One rank's share of a sequence-sharded LM head: its tokens' losses
    and dH rows, the dW summed over every shard, and the job's total (summed) loss."""

    loss: torch.Tensor  # this shard's per-token nats
    dh: torch.Tensor  # this shard's rows
    dw: torch.Tensor  # [V, D], all-reduced: identical on every rank
    total_loss: float  # sum over all shards' tokens (oracle.py:129-133 sums, never averages)
    peak_aux_elements: int


def sharded_fused_lmhead_loss(h_local: torch.Tensor, w_head: torch.Tensor, targets_local: torch.Tensor,
                              cfg: FusionConfig, group=None) -> ShardedLossResult:
    """The LM head of a sequence sharded over the ranks of ``group`` (one process per GPU, W
    replicated): each rank runs the fused head on its own tokens, then dW is summed over the
    shards (all_reduce_dw) and the per-token losses are summed into the job's loss.  Token
    shards are independent in the forward and in dH (lmhead.py:41-93 is row-separable), so the
    only exchange is dW and one scalar."""
    import torch.distributed as dist

    v, d = w_head.shape
    dev = h_local.device
    dw = torch.zeros(v, max(8, (d + 7) // 8 * 8), dtype=torch.float32, device=dev)
    res = fused_lmhead_loss(h_local, w_head, targets_local, cfg, device=dev, dw_out=dw)
    total = res.loss.double().sum().reshape(1)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(total, group=group)
    all_reduce_dw(dw, group)
    return ShardedLossResult(loss=res.loss, dh=res.dh, dw=dw[:, :d], total_loss=float(total.item()),
                             peak_aux_elements=res.peak_aux_elements)


def memory_footprint(n: int, vocab: int, dim: int, cfg: FusionConfig) -> tuple[int, int]:
    """(naive N*V, fused min(B_s, N)*V) logits-class elements (lmhead.py:96-110)."""
    if n < 1 or vocab < 1 or dim < 1:
        raise ValueError("n, vocab, dim must all be >= 1")
    return n * vocab, min(cfg.rows_per_tile, n) * vocab


def tile_working_set(n: int, vocab: int, dim: int, cfg: FusionConfig) -> int:
    """Per-tile scratch beyond the retained logits (lmhead.py:113-116)."""
    bs, bv = min(cfg.rows_per_tile, n), min(cfg.vocab_per_tile, vocab)
    return bs * dim + bv * dim + 4 * bs
