"""Token-to-device layouts and exact workload accounting.

Public surface of ``burstsim.partitioning`` (partitioning.py:38-250) with the
same 1-based conventions and ValueError messages.  Differences are internal:
token ids are produced by vectorised closed forms (the same formulas the
kernels evaluate in csrc/bb_mask.cuh::token_id), and pair counts use sorted-id
searches instead of dense n x n matrices, so ``balance_report`` and
``global_unmasked_pairs`` stay exact and cheap at 1M tokens.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .masks import BLOCK_SPARSE, CAUSAL, FULL, SLIDING_WINDOW, MaskSpec, allowed_pairs, block_sparse_mask, validate_mask

CONTIGUOUS = "contiguous"
ZIGZAG = "zigzag"
STRIPED = "striped"
BLOCK_STRIPED = "block_striped"
LAYOUT_KINDS = (CONTIGUOUS, ZIGZAG, STRIPED, BLOCK_STRIPED)


@dataclass(frozen=True)
class Shard:
    device: int  # 1-based
    token_ids: tuple[int, ...]


@dataclass(frozen=True)
class ShardLayout:
    """kind x N x G (+ block_len); divisibility rules of partitioning.py:53-72."""

    kind: str
    seq_len: int
    devices: int
    block_len: int | None = None

    def __post_init__(self):
        if self.kind not in LAYOUT_KINDS:
            raise ValueError(f"unknown layout kind {self.kind!r}, expected {LAYOUT_KINDS}")
        n, g = self.seq_len, self.devices
        if n < 1 or g < 1:
            raise ValueError(f"need seq_len >= 1 and devices >= 1, got N={n}, G={g}")
        if self.kind in (CONTIGUOUS, STRIPED) and n % g:
            raise ValueError(f"{self.kind} layout needs G | N, got N={n}, G={g}")
        if self.kind == ZIGZAG and n % (2 * g):
            raise ValueError(f"zigzag layout needs 2G | N, got N={n}, G={g}")
        if self.kind == BLOCK_STRIPED:
            if self.block_len is None:
                raise ValueError("block_striped layout needs block_len")
            if self.block_len % g:
                raise ValueError(f"block_striped needs G | block_len, got block_len={self.block_len}, G={g}")
            if n % self.block_len:
                raise ValueError(f"block_striped needs block_len | N, got N={n}, block_len={self.block_len}")

    @property
    def shard_size(self) -> int:
        return self.seq_len // self.devices


def device_token_ids(layout: ShardLayout, device: int) -> np.ndarray:
    """Increasing 1-based global ids owned by 1-based ``device`` (shard row order)."""
    n, g = layout.seq_len, layout.devices
    r = np.arange(layout.shard_size, dtype=np.int64)
    if layout.kind == CONTIGUOUS:
        return (device - 1) * (n // g) + r + 1
    if layout.kind == ZIGZAG:
        p = n // (2 * g)
        return np.where(r < p, (device - 1) * p + r + 1, n - device * p + (r - p) + 1)
    if layout.kind == STRIPED:
        return device + g * r
    per = layout.block_len // g
    return (r // per) * layout.block_len + (r % per) * g + device


def make_layout(kind: str, seq_len: int, devices: int, block_len: int | None = None) -> list[Shard]:
    return layout_shards(ShardLayout(kind, seq_len, devices, block_len))


def layout_shards(layout: ShardLayout) -> list[Shard]:
    return [
        Shard(dev, tuple(int(t) for t in device_token_ids(layout, dev))) for dev in range(1, layout.devices + 1)
    ]


def shard_token_arrays(layout: ShardLayout) -> list[np.ndarray]:
    return [device_token_ids(layout, dev) for dev in range(1, layout.devices + 1)]


def local_pair_mask(layout: ShardLayout, mask: MaskSpec, i: int, j: int, use_closed_form: bool = True) -> np.ndarray:
    """Allowed (local query of device i, local key of device j) pairs (partitioning.py:120-169)."""
    g = layout.devices
    if not (1 <= i <= g and 1 <= j <= g):
        raise ValueError(f"device indices must lie in [1, {g}], got i={i}, j={j}")
    validate_mask(mask, layout.seq_len)
    if use_closed_form and mask.kind == CAUSAL and layout.kind in (ZIGZAG, STRIPED):
        size = layout.shard_size
        if layout.kind == ZIGZAG:
            half = size // 2
            if i == j:
                ids = device_token_ids(layout, i)
                return ids[None, :] <= ids[:, None]
            out = np.zeros((size, size), dtype=bool)
            if i < j:
                out[half:, :] = True  # back-block queries see all of device j
            else:
                out[:, :half] = True  # all queries see device j's front block
            return out
        a = np.arange(size)
        return a[None, :] <= a[:, None] if i >= j else a[None, :] < a[:, None]
    return allowed_pairs(mask, device_token_ids(layout, i), device_token_ids(layout, j))


def local_pair_set(layout: ShardLayout, mask: MaskSpec, i: int, j: int, use_closed_form: bool = True):
    qs, ks = np.nonzero(local_pair_mask(layout, mask, i, j, use_closed_form))
    return frozenset((int(a) + 1, int(b) + 1) for a, b in zip(qs, ks))


def pair_count(mask: MaskSpec, q_ids: np.ndarray, k_ids: np.ndarray) -> int:
    """sum(allowed_pairs(mask, q_ids, k_ids)) without the matrix; k_ids sorted ascending."""
    q = np.asarray(q_ids, dtype=np.int64)
    k = np.asarray(k_ids, dtype=np.int64)
    if mask.kind == FULL:
        return int(q.size * k.size)
    if mask.kind == CAUSAL:
        return int(np.searchsorted(k, q, side="right").sum())
    if mask.kind == SLIDING_WINDOW:
        hi = np.searchsorted(k, q, side="right")
        lo = np.searchsorted(k, q - mask.window, side="right")
        return int((hi - lo).sum())
    if mask.kind == BLOCK_SPARSE:
        bl = int(mask.block_len)
        nb = mask.block_mask.shape[0]
        kb = np.bincount((k - 1) // bl, minlength=nb)  # keys per block
        qb = np.bincount((q - 1) // bl, minlength=nb)  # queries per block
        return int(qb @ mask.block_mask @ kb)
    raise ValueError(f"unknown mask kind {mask.kind!r}")


@dataclass(frozen=True)
class WorkloadReport:
    per_device_pairs: tuple[int, ...]
    per_step_pairs: tuple[tuple[int, ...], ...]  # [device][ring step]
    total_pairs: int

    @property
    def device_spread(self) -> int:
        return max(self.per_device_pairs) - min(self.per_device_pairs)

    def step_spread(self, step: int) -> int:
        col = [row[step] for row in self.per_step_pairs]
        return max(col) - min(col)

    @property
    def max_step_spread(self) -> int:
        return max(self.step_spread(t) for t in range(len(self.per_step_pairs[0])))


def pair_count_matrix(layout: ShardLayout, mask: MaskSpec) -> np.ndarray:
    """counts[i-1, j-1] = allowed pairs between query device i and key device j."""
    validate_mask(mask, layout.seq_len)
    g = layout.devices
    ids = shard_token_arrays(layout)
    out = np.zeros((g, g), dtype=np.int64)
    for i in range(g):
        for j in range(g):
            out[i, j] = pair_count(mask, ids[i], ids[j])
    return out


def balance_report(layout: ShardLayout, mask: MaskSpec) -> WorkloadReport:
    """Per-device / per-ring-step pair counts; step t pairs device i with shard (i-1-t) mod G
    (partitioning.py:205-225)."""
    counts = pair_count_matrix(layout, mask)
    g = layout.devices
    per_step = tuple(tuple(int(counts[i, (i - 1 - t) % g]) for t in range(g)) for i in range(g))
    return WorkloadReport(
        per_device_pairs=tuple(int(x) for x in counts.sum(axis=1)),
        per_step_pairs=per_step,
        total_pairs=int(counts.sum()),
    )


def global_unmasked_pairs(mask: MaskSpec, seq_len: int) -> int:
    validate_mask(mask, seq_len)
    ids = np.arange(1, seq_len + 1, dtype=np.int64)
    return pair_count(mask, ids, ids)


def block_mask_from_window(seq_len: int, block_len: int, window: int) -> MaskSpec:
    """Causal band of width window/block_len blocks (partitioning.py:235-250)."""
    if block_len < 1 or seq_len % block_len:
        raise ValueError(f"block_len {block_len} must divide seq_len {seq_len}")
    if window < 1 or window % block_len:
        raise ValueError(f"window {window} must be a positive multiple of block_len {block_len}")
    side = seq_len // block_len
    gap = np.arange(side)[:, None] - np.arange(side)[None, :]
    return block_sparse_mask(((gap >= 0) & (gap < window // block_len)).astype(np.int64), block_len)
