"""Golden vectors for a cfg4-shaped case, by running the REFERENCE itself (burstsim, read-only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cfg4_golden.py

cfg4 (BASELINE.json) is GQA 32q/8kv + a 32K sliding window + documents over 512K tokens in the
block_striped layout.  The reference has no document mask and no heads, but it runs any
block_sparse mask (masks.py:55-61) in any layout, single head.  This script scales cfg4 down
to N=1024 over G=4 (block_striped, layout block 64): mask blocks of 32 tokens, the block band
of a 256-token window (partitioning.block_mask_from_window) AND two causal 512-token documents
-- the same block-level structure bench.py's swa_doc mask has -- and runs distributed_forward,
burst_backward and ring_backward for two query heads that share one K/V head (seeds differ per
query head; inputs are regenerated from their seeds, numerics.py:95-98).  GQA is then pinned through the reference too: the engine's dK/dV for the shared
head must equal the sum of the two single-head reference runs.

Writes tests/golden/golden_cfg4_fp64.npz (float64).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from burstsim import distributed, fabric, masks, numerics, partitioning  # noqa: E402

OUT = Path(__file__).resolve().parent
N, G, D, LAYOUT_BLOCK = 1024, 4, 16, 64
MASK_BLOCK, WINDOW, DOC = 32, 256, 512
QHEADS = 2


def doc_block_mask(n: int, block: int, doc: int) -> np.ndarray:
    """Block-level causal documents: block (i, j) allowed iff same document and j <= i."""
    nb = n // block
    doc_of = np.arange(nb) * block // doc
    i, j = np.meshgrid(np.arange(nb), np.arange(nb), indexing="ij")
    return ((doc_of[i] == doc_of[j]) & (j <= i)).astype(np.int64)


def main():
    band = partitioning.block_mask_from_window(N, MASK_BLOCK, WINDOW).block_mask
    bm = np.logical_and(band, doc_block_mask(N, MASK_BLOCK, DOC)).astype(np.int64)
    mask = masks.block_sparse_mask(bm, MASK_BLOCK)
    lay = partitioning.ShardLayout("block_striped", N, G, block_len=LAYOUT_BLOCK)
    topo = fabric.Topology(1, G)
    F = {"block_mask": bm, "meta": np.array([N, G, D, LAYOUT_BLOCK, MASK_BLOCK, WINDOW, DOC, QHEADS])}
    k = numerics.seeded_random_matrix(N, D, 4001)
    v = numerics.seeded_random_matrix(N, D, 4002)
    gr = lambda arrs: distributed.gather_rows(lay, arrs)  # noqa: E731
    for h in range(QHEADS):
        q = numerics.seeded_random_matrix(N, D, 4010 + h)
        do = numerics.seeded_random_matrix(N, D, 4020 + h)
        st = distributed.make_device_states(lay, q, k, v)
        distributed.distributed_forward(st, lay, mask, topo)
        do_sh = distributed.shard_rows(lay, do)
        distributed.burst_backward(st, do_sh, lay, mask, topo)
        st2 = distributed.make_device_states(lay, q, k, v)
        distributed.distributed_forward(st2, lay, mask, topo)
        distributed.ring_backward(st2, do_sh, lay, mask, topo)
        F[f"o{h}"] = gr([s.o for s in st])
        F[f"lse{h}"] = gr([s.lse for s in st])
        F[f"dq{h}"] = gr([s.dq for s in st])
        F[f"dk{h}"] = gr([s.dk for s in st])
        F[f"dv{h}"] = gr([s.dv for s in st])
        if h == 0:  # the K/V-circulating backward once (the reference pins burst == ring to 1e-10)
            F["ring_dq0"] = gr([s.dq for s in st2])
            F["ring_dk0"] = gr([s.dk for s in st2])
            F["ring_dv0"] = gr([s.dv for s in st2])
    np.savez_compressed(OUT / "golden_cfg4_fp64.npz", **F)
    print(f"wrote {OUT / 'golden_cfg4_fp64.npz'}: mask density {bm.mean():.3f}")


if __name__ == "__main__":
    main()
