"""Bit-exact checks of the masks the kernels realise on the device.

The reference builds dense local pair masks (partitioning.py:120-169, local_pair_mask); the
kernels never do -- they classify 128x128 tiles from token-id bounds (skip / full / partial,
bb_mask.cuh classify_tile), bound each CTA's range with a binary search (active_runs) and
evaluate the predicate per element only on partial tiles (row_mask_bits).  These tests pin
that realisation to local_pair_mask for every (query device, key device) pair, 4 layouts x
{full, causal, sliding window, block-sparse band, document} x N in {256, 1000 (ragged
tiles), 4096}, three ways:

1. bb_debug_mask_tiles dumps the classes and element mask each kernel applies (same device
   functions, same arguments); the element mask must equal local_pair_mask exactly, every
   SKIP tile must be empty, every FULL tile full, and the classes must equal a host
   restatement of classify_tile wherever the CTA range search did not already skip the tile.
2. The forward kernel itself with Q = K = 0 (every allowed score 0, so P = 1 exactly) and V
   one-hot (columns 0-63: key index mod 64, columns 64-127: key index div 64): exp(lse) must
   be the row's allowed-key count and O * count the per-class counts, as integers.
3. The backward kernel with Q = K = V = 0, lse = 0, D = 0 and dO one-hot the same way over
   query indices: dV must hold the exact per-class allowed-query counts of every key row,
   dK and dQ must be exactly zero.
"""

import math

import numpy as np
import pytest
import torch

import paper_2509_19836_b200 as bb
from paper_2509_19836_b200 import kernels as K
from paper_2509_19836_b200.partitioning import device_token_ids

pytestmark = pytest.mark.gpu

G = 4
LAYOUTS = ("contiguous", "zigzag", "striped", "block_striped")
MASKS = ("full", "causal", "window", "block", "doc")
SKIP, FULL, PARTIAL = 0, 1, 2


def _block_len(n):
    return {256: 16, 1000: 8, 4096: 64}[n]


def make_case(kind, n, mname):
    bl = _block_len(n)
    layout = bb.ShardLayout(kind, n, G, bl if kind == "block_striped" else None)
    if mname == "full":
        mask = bb.full_mask()
    elif mname == "causal":
        mask = bb.causal_mask()
    elif mname == "window":
        mask = bb.sliding_window_mask(n // 3 + 7)  # not tile-aligned: partial tiles on both edges
    elif mname == "block":
        mask = bb.block_mask_from_window(n, bl, bl * (n // bl // 3))
    else:
        nb = n // bl
        mask = bb.document_mask([bl * (nb - 2 * (nb // 4)), bl * (nb // 4), bl * (nb // 4)], block_len=bl)
    return layout, mask


# ---- host restatement of classify_tile (bb_mask.cuh), for the class comparison -------------
def host_tile_class(mask, q_ids, k_ids, full_width):
    qa, qb, ka, kb = int(q_ids[0]), int(q_ids[-1]), int(k_ids[0]), int(k_ids[-1])
    cls = PARTIAL
    if mask.kind == "full":
        cls = FULL
    elif mask.kind == "causal":
        if ka > qb:
            return SKIP
        if kb <= qa:
            cls = FULL
    elif mask.kind == "sliding_window":
        w = mask.window
        if ka > qb or qa - kb >= w:
            return SKIP
        if kb <= qa and qb - ka < w:
            cls = FULL
    else:
        bl = mask.block_len
        qb0, qb1, kb0, kb1 = (qa - 1) // bl, (qb - 1) // bl, (ka - 1) // bl, (kb - 1) // bl
        if (qb1 - qb0 + 1) * (kb1 - kb0 + 1) <= 256:
            sub = np.asarray(mask.block_mask)[qb0:qb1 + 1, kb0:kb1 + 1] != 0
            if not sub.any():
                return SKIP
            if sub.all():
                cls = FULL
    if cls == FULL and not full_width:
        cls = PARTIAL
    return cls


@pytest.mark.parametrize("n", [256, 1000, 4096])
@pytest.mark.parametrize("kind", LAYOUTS)
@pytest.mark.parametrize("mname", MASKS)
def test_kernel_mask_realisation_is_local_pair_mask(cuda, n, kind, mname):
    layout, mask = make_case(kind, n, mname)
    dev = torch.device("cuda:0")
    dm = K.device_mask(mask, dev)
    m = layout.shard_size
    conservative = 0
    for view in ("fwd", "bwd"):
        for i in range(1, G + 1):
            for j in range(1, G + 1):
                cls, allowed = K.debug_mask_tiles(layout, dm, i, j, m, m, view, dev)
                ref = bb.local_pair_mask(layout, mask, i, j)
                assert np.array_equal(allowed, ref), (view, i, j, int((allowed != ref).sum()))
                qi, ki = device_token_ids(layout, i), device_token_ids(layout, j)
                for qt in range(cls.shape[0]):
                    for kt in range(cls.shape[1]):
                        sub = ref[qt * 128:(qt + 1) * 128, kt * 128:(kt + 1) * 128]
                        c = int(cls[qt, kt])
                        if c == SKIP:
                            assert not sub.any(), (view, i, j, qt, kt)
                            continue
                        if c == FULL:
                            assert sub.all(), (view, i, j, qt, kt)
                        hc = host_tile_class(mask, qi[qt * 128:(qt + 1) * 128], ki[kt * 128:(kt + 1) * 128],
                                             min(m - kt * 128, 128) == 128)
                        assert c == hc, (view, i, j, qt, kt, c, hc)
                        conservative += c == PARTIAL and (sub.all() or not sub.any())
    # (partial tiles that turn out uniform, e.g. a zigzag tile straddling its shard's two
    # halves, cost time, never correctness: `conservative` counts them for debugging)


def _onehot_rows(rows, d=128):
    """[rows, d] one-hot codes: column r % 64 and column 64 + r // 64 (needs rows <= 4096)."""
    x = np.zeros((rows, d), dtype=np.float32)
    r = np.arange(rows)
    x[r, r % 64] = 1
    x[r, 64 + r // 64] = 1
    return x


def _class_counts(ref):
    """Per row of a bool [a, b] matrix: counts of allowed columns by c % 64 and c // 64."""
    cols = np.arange(ref.shape[1])
    out = np.zeros((ref.shape[0], 128), dtype=np.int64)
    for c in range(64):
        out[:, c] = ref[:, cols % 64 == c].sum(1)
    for t in range(-(-ref.shape[1] // 64)):
        out[:, 64 + t] = ref[:, cols // 64 == t].sum(1)
    return out


@pytest.mark.parametrize("n", [1000, 4096])
@pytest.mark.parametrize("kind", LAYOUTS)
@pytest.mark.parametrize("mname", MASKS)
def test_forward_kernel_counts_allowed_keys_exactly(cuda, n, kind, mname):
    layout, mask = make_case(kind, n, mname)
    dev = torch.device("cuda:0")
    dm = K.device_mask(mask, dev)
    m = layout.shard_size
    zeros = torch.zeros(m, 1, 128, dtype=torch.bfloat16, device=dev)
    v = torch.from_numpy(_onehot_rows(m)).to(torch.bfloat16).view(m, 1, 128).to(dev)
    for i in range(1, G + 1):
        for j in range(1, G + 1):
            o = torch.zeros(m, 1, 128, device=dev)
            lse = torch.full((1, m), float("-inf"), device=dev)
            K.attn_fwd_step(zeros, zeros, v, o, lse, layout, dm, i, j, 1 / math.sqrt(128))
            ref = bb.local_pair_mask(layout, mask, i, j)
            count = ref.sum(1)
            lse_h = lse[0].double().cpu().numpy()
            o_h = o[:, 0].double().cpu().numpy()
            none = count == 0
            assert np.all(np.isneginf(lse_h[none])) and not np.any(o_h[none]), (i, j)
            got = np.rint(np.exp(lse_h[~none])).astype(np.int64)
            assert np.array_equal(got, count[~none]), (i, j)
            cc = np.rint(o_h[~none] * count[~none, None]).astype(np.int64)
            assert np.array_equal(cc, _class_counts(ref)[~none]), (i, j)


@pytest.mark.parametrize("n", [1000, 4096])
@pytest.mark.parametrize("kind", LAYOUTS)
@pytest.mark.parametrize("mname", MASKS)
def test_backward_kernel_counts_allowed_queries_exactly(cuda, n, kind, mname):
    layout, mask = make_case(kind, n, mname)
    dev = torch.device("cuda:0")
    dm = K.device_mask(mask, dev)
    m = layout.shard_size
    zeros = torch.zeros(m, 1, 128, dtype=torch.bfloat16, device=dev)
    do = torch.from_numpy(_onehot_rows(m)).to(torch.bfloat16).view(m, 1, 128).to(dev)
    lse = torch.zeros(1, m, device=dev)
    delta = torch.zeros(1, m, device=dev)
    for i in range(1, G + 1):
        for j in range(1, G + 1):
            dq = torch.zeros(m, 1, 128, device=dev)
            dk = torch.zeros(m, 1, 128, device=dev)
            dv = torch.zeros(m, 1, 128, device=dev)
            K.attn_bwd_step(zeros, zeros, zeros, do, lse, delta, dq, dk, dv, layout, dm, i, j, 1 / math.sqrt(128))
            ref = bb.local_pair_mask(layout, mask, i, j)
            got = np.rint(dv[:, 0].double().cpu().numpy()).astype(np.int64)
            assert np.array_equal(got, _class_counts(ref.T)), (i, j)
            assert not dk.any() and not dq.any(), (i, j)
