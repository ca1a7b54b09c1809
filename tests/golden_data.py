"""Loader for the golden vectors produced by running the reference (tests/golden/make_golden.py)."""

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=1)
def meta() -> dict:
    return json.loads((GOLDEN / "golden.json").read_text())


@lru_cache(maxsize=1)
def arrays():
    return np.load(GOLDEN / "golden_fp64.npz")


def oracle_mask(desc: dict) -> tuple:
    """golden mask description -> oracle mask tuple (kind, window, block_len, block_mask)."""
    bm = None if desc["block_mask"] is None else np.asarray(desc["block_mask"], dtype=np.int64)
    return (desc["kind"], desc["window"], desc["block_len"], bm)


def product_mask(desc: dict):
    from paper_2509_19836_b200 import masks as M

    if desc["kind"] == "full":
        return M.full_mask()
    if desc["kind"] == "causal":
        return M.causal_mask()
    if desc["kind"] == "sliding_window":
        return M.sliding_window_mask(desc["window"])
    return M.block_sparse_mask(np.asarray(desc["block_mask"]), desc["block_len"])


def unpack_pairs(key: str, g: int, n: int) -> np.ndarray:
    """[G*G, n/G, n/G] bool stack of local pair masks (i-major, j-minor)."""
    size = n // g
    return np.unpackbits(arrays()[key], axis=-1, count=size).astype(bool)


def cfg4_golden():
    """tests/golden/golden_cfg4_fp64.npz (make_cfg4_golden.py: burstsim on a cfg4-shaped case),
    with the inputs regenerated from their seeds: (arrays, N, G, D, layout block, mask block, Hq)."""
    from oracle import burst_oracle as O

    A = dict(np.load(GOLDEN / "golden_cfg4_fp64.npz"))
    n, g, d, lb, mb, _w, _doc, hq = (int(x) for x in A["meta"])
    A["k"] = O.seeded_random_matrix(n, d, 4001)[:, None]
    A["v"] = O.seeded_random_matrix(n, d, 4002)[:, None]
    A["q"] = np.stack([O.seeded_random_matrix(n, d, 4010 + h) for h in range(hq)], axis=1)
    A["do"] = np.stack([O.seeded_random_matrix(n, d, 4020 + h) for h in range(hq)], axis=1)
    return A, n, g, d, lb, mb, hq
