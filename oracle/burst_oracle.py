"""CPU oracle for the BurstAttention hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in float64 NumPy, the reference algorithm of
``burstsim`` (/root/reference/pkg/src/burstsim, arXiv 2509.19836's desk-scale
library).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it, and only as the
checker or the timed CPU baseline.  The product path (paper_2509_19836_b200/)
never imports it; it runs the sm_100a kernels or raises.

Pinning: every function below is checked against golden vectors produced by
running the reference itself (tests/golden/make_golden.py -> *.npz/*.json) and
against the known-answer values in the reference's own tests
(tests/test_oracle_golden.py).  Parity status: pinned.

Each function cites the reference file:line it follows.  The algorithms are the
reference's; the code is organised differently (multi-head drivers, explicit
loops over ring steps), so it can also serve as the CPU baseline the bench
times ("kind": "port").
"""

from __future__ import annotations

import math

import numpy as np

NEG_INF = -np.inf

# ----------------------------------------------------------------- numerics
# numerics.py:35-45 -- every product through einsum(optimize=False): fixed order, no BLAS.


def mm(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    return np.einsum("ik,kj->ij", a, b, optimize=False)


def lse_rows(s: np.ndarray) -> np.ndarray:
    """numerics.py:48-59: max-shifted row LSE; an all -inf row gives -inf."""
    m = s.max(axis=1)
    out = np.full(s.shape[0], NEG_INF)
    live = m != NEG_INF
    if live.any():
        out[live] = m[live] + np.log(np.exp(s[live] - m[live, None]).sum(axis=1))
    return out


def lse_merge(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """numerics.py:62-69: np.logaddexp keeps -inf as the exact identity."""
    return np.logaddexp(a, b)


def exp_shifted(s: np.ndarray, lse: np.ndarray) -> np.ndarray:
    """numerics.py:101-107: exp(s - lse) with -inf rows giving exact zeros."""
    out = np.zeros_like(s)
    live = lse != NEG_INF
    out[live] = np.exp(s[live] - lse[live, None])
    return out


def exp_gap(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """numerics.py:110-116: exp(a - b) with exp(-inf - x) == 0."""
    out = np.zeros_like(a)
    live = a != NEG_INF
    out[live] = np.exp(a[live] - b[live])
    return out


def rowsum_hadamard(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """numerics.py:86-92."""
    return np.einsum("ij,ij->i", a, b, optimize=False)


def seeded_random_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """numerics.py:95-98: PCG64 uniform in [-1, 1]."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(rows, cols))


# ----------------------------------------------------------------- masks / layouts
# masks.py:89-104 predicates on 1-based ids; mask = (kind, window, block_len, block_mask)


def allowed(mask: tuple, q_ids, k_ids) -> np.ndarray:
    kind, window, block_len, block_mask = mask
    q = np.asarray(q_ids, dtype=np.int64).reshape(-1, 1)
    k = np.asarray(k_ids, dtype=np.int64).reshape(1, -1)
    if kind == "full":
        return np.ones((q.shape[0], k.shape[1]), dtype=bool)
    if kind == "causal":
        return k <= q
    if kind == "sliding_window":
        return (q - k >= 0) & (q - k < window)
    if kind == "block_sparse":
        return np.asarray(block_mask)[(q - 1) // block_len, (k - 1) // block_len] == 1
    raise ValueError(kind)


def shard_ids(kind: str, n: int, g: int, block_len: int | None = None) -> list[np.ndarray]:
    """partitioning.py:85-112, literal loops over devices and positions."""
    out = []
    for dev in range(1, g + 1):
        if kind == "contiguous":
            p = n // g
            ids = list(range((dev - 1) * p + 1, dev * p + 1))
        elif kind == "zigzag":
            p = n // (2 * g)
            ids = list(range((dev - 1) * p + 1, dev * p + 1)) + list(range(n - dev * p + 1, n - (dev - 1) * p + 1))
        elif kind == "striped":
            ids = [dev + g * m for m in range(n // g)]
        elif kind == "block_striped":
            ids = [b * block_len + pos + 1 for b in range(n // block_len) for pos in range(block_len) if pos % g == dev - 1]
        else:
            raise ValueError(kind)
        out.append(np.asarray(ids, dtype=np.int64))
    return out


def local_allowed(kind: str, n: int, g: int, block_len, mask: tuple, i: int, j: int) -> np.ndarray:
    """partitioning.py:120-169 (the closed forms equal the general predicate, :136-144)."""
    ids = shard_ids(kind, n, g, block_len)
    return allowed(mask, ids[i - 1], ids[j - 1])


def ring_visit(num_nodes: int, gpus_per_node: int) -> list[list[int]]:
    """fabric.py:122-139 / :184-201: 0-based shard visited by each device at each step."""
    g = num_nodes * gpus_per_node
    if g == 1:
        return [[0]]
    if num_nodes == 1:
        return [[(dev - t - 1) % g for t in range(g)] for dev in range(g)]
    rows = []
    for dev in range(g):
        node, slot = divmod(dev, gpus_per_node)
        rows.append(
            [((node - a) % num_nodes) * gpus_per_node + (slot - b) % gpus_per_node for a in range(num_nodes) for b in range(gpus_per_node)]
        )
    return rows


# ----------------------------------------------------------------- full-materialisation oracle


def attention_forward(q, k, v, mask_full: np.ndarray):
    """oracle.py:80-95 with a precomputed dense allowed matrix."""
    s = np.where(mask_full, mm(q, k.T) / np.sqrt(q.shape[1]), NEG_INF)
    lse = lse_rows(s)
    if np.any(lse == NEG_INF):
        raise ValueError(f"query row {int(np.argmax(lse == NEG_INF)) + 1} has no unmasked key")
    return mm(exp_shifted(s, lse), v), lse


def attention_backward(q, k, v, o, lse, do, mask_full: np.ndarray):
    """oracle.py:98-119: dP = dO V^T, D = rowsum(dO o O), dS = P o (dP - D)."""
    scale = 1.0 / np.sqrt(q.shape[1])
    s = np.where(mask_full, mm(q, k.T) / np.sqrt(q.shape[1]), NEG_INF)
    p = exp_shifted(s, lse)
    ds = p * (mm(do, v.T) - rowsum_hadamard(do, o)[:, None])
    return mm(ds, k) * scale, mm(ds.T, q) * scale, mm(p.T, do)


# ----------------------------------------------------------------- ring passes (single head)


def ring_forward(qs, ks, vs, pair_mask, visit):
    """distributed.py:151-195.  qs/ks/vs: per-device shards; pair_mask(i, j) -> bool [n, n]
    (0-based devices); visit[i][t] = 0-based shard device i folds in at step t.
    Returns per-device (O, lse)."""
    g = len(qs)
    scale = 1.0 / np.sqrt(qs[0].shape[1])
    o = [np.zeros_like(x) for x in qs]
    lse = [np.full(x.shape[0], NEG_INF) for x in qs]
    for t in range(g):
        for i in range(g):
            j = visit[i][t]
            am = pair_mask(i, j)
            if not am.any():
                continue  # compute skipped, transfer still counted (:178-179)
            s = np.where(am, mm(qs[i], ks[j].T) * scale, NEG_INF)
            l_step = lse_rows(s)
            o_step = mm(exp_shifted(s, l_step), vs[j])
            l_new = lse_merge(lse[i], l_step)
            o[i] = exp_gap(l_step, l_new)[:, None] * o_step + exp_gap(lse[i], l_new)[:, None] * o[i]
            lse[i] = l_new
    for i in range(g):
        if np.any(lse[i] == NEG_INF):
            row = int(np.argmax(lse[i] == NEG_INF)) + 1
            raise ValueError(f"device {i + 1} query row {row} has no unmasked key globally")
    return o, lse


def burst_backward(qs, ks, vs, os_, lses, dos, pair_mask, visit):
    """distributed.py:255-299: K/V stationary, (Q, dQ, dO, D, lse) circulate; D once (:274-275)."""
    g = len(qs)
    scale = 1.0 / np.sqrt(qs[0].shape[1])
    d_vec = [rowsum_hadamard(dos[i], os_[i]) for i in range(g)]
    dk = [np.zeros_like(x) for x in ks]
    dv = [np.zeros_like(x) for x in vs]
    dq = [np.zeros_like(x) for x in qs]  # payload dQ, indexed by owner
    for t in range(g):
        for i in range(g):
            j = visit[i][t]  # device i holds query payload of shard j
            am = pair_mask(j, i)
            if not am.any():
                continue
            s = np.where(am, mm(qs[j], ks[i].T) * scale, NEG_INF)
            p = exp_shifted(s, lses[j])
            dv[i] += mm(p.T, dos[j])
            ds = p * (mm(dos[j], vs[i].T) - d_vec[j][:, None])
            dk[i] += mm(ds.T, qs[j]) * scale
            dq[j] += mm(ds, ks[i]) * scale
    return dq, dk, dv, d_vec


def ring_backward(qs, ks, vs, os_, lses, dos, pair_mask, visit):
    """distributed.py:207-252: K, V, dK, dV circulate; dQ local; D recomputed per step (:244)."""
    g = len(qs)
    scale = 1.0 / np.sqrt(qs[0].shape[1])
    dk = [np.zeros_like(x) for x in ks]
    dv = [np.zeros_like(x) for x in vs]
    dq = [np.zeros_like(x) for x in qs]
    for t in range(g):
        for i in range(g):
            j = visit[i][t]
            am = pair_mask(i, j)
            if not am.any():
                continue
            s = np.where(am, mm(qs[i], ks[j].T) * scale, NEG_INF)
            p = exp_shifted(s, lses[i])
            dv[j] += mm(p.T, dos[i])
            ds = p * (mm(dos[i], vs[j].T) - rowsum_hadamard(dos[i], os_[i])[:, None])
            dk[j] += mm(ds.T, qs[i]) * scale
            dq[i] += mm(ds, ks[j]) * scale
    return dq, dk, dv


# ----------------------------------------------------------------- multi-head / GQA drivers
# The reference is single-head; heads are independent, GQA repeats K/V
# head h*Hkv//Hq and sums dK/dV over the group (parity unpinned for GQA).


def mh_ring_attention(q, k, v, do, layout: tuple, mask: tuple, visit, backward: str | None = "burst"):
    """q,do: [N, Hq, d]; k,v: [N, Hkv, d] in GLOBAL token order.  layout = (kind, N, G, block_len).
    Returns dict of global-order O [N,Hq,d], lse [Hq,N] and (if backward) dQ, dK, dV."""
    kind, n, g, bl = layout
    ids = shard_ids(kind, n, g, bl)
    rows = [x - 1 for x in ids]
    masks = {(i, j): allowed(mask, ids[i], ids[j]) for i in range(g) for j in range(g)}
    pm = lambda i, j: masks[(i, j)]  # noqa: E731
    hq, hkv = q.shape[1], k.shape[1]
    rep = hq // hkv
    out = {"o": np.zeros(q.shape), "lse": np.zeros((hq, n))}
    if backward:
        out.update(dq=np.zeros(q.shape), dk=np.zeros(k.shape), dv=np.zeros(v.shape))
    for h in range(hq):
        hk = h // rep
        qs = [q[r, h] for r in rows]
        ks = [k[r, hk] for r in rows]
        vs = [v[r, hk] for r in rows]
        o, lse = ring_forward(qs, ks, vs, pm, visit)
        for r, oi, li in zip(rows, o, lse):
            out["o"][r, h] = oi
            out["lse"][h, r] = li
        if backward:
            dos = [do[r, h] for r in rows]
            fn = burst_backward if backward == "burst" else ring_backward
            res = fn(qs, ks, vs, o, lse, dos, pm, visit)
            for r, a, b, c in zip(rows, res[0], res[1], res[2]):
                out["dq"][r, h] = a
                out["dk"][r, hk] += b
                out["dv"][r, hk] += c
    return out


# ----------------------------------------------------------------- accounting


def comm_elements(pass_kind: str, n: int, d: int, g: int) -> int:
    """fabric.py:306-321: 2Nd / 4Nd / 3Nd+2N per device per pass."""
    return {"forward": 2 * n * d, "ring_backward": 4 * n * d, "burst_backward": 3 * n * d + 2 * n}[pass_kind]


def balance_counts(kind, n, g, block_len, mask):
    """partitioning.py:205-225: per-device totals and per-step counts (step t -> shard (i-1-t) mod G)."""
    counts = np.array([[local_allowed(kind, n, g, block_len, mask, i, j).sum() for j in range(1, g + 1)] for i in range(1, g + 1)])
    per_step = [[int(counts[i, (i - 1 - t) % g]) for t in range(g)] for i in range(g)]
    return [int(x) for x in counts.sum(1)], per_step, int(counts.sum())


# ----------------------------------------------------------------- LM head


def naive_lmhead(h, w, y):
    """oracle.py:129-154: full logits, sum-reduced CE, dlogits = softmax - onehot."""
    logits = mm(h, w.T)
    lse = lse_rows(logits)
    rows = np.arange(h.shape[0])
    loss = lse - logits[rows, y]
    g = exp_shifted(logits, lse)
    g[rows, y] -= 1.0
    return loss, mm(g, w), mm(g.T, h)


def fused_lmhead(h, w, y, rows_per_tile: int, vocab_per_tile: int):
    """lmhead.py:41-93: row tiles x vocab tiles, streaming LSE, logits retained per row tile."""
    n, _ = h.shape
    v = w.shape[0]
    loss = np.zeros(n)
    dh = np.zeros_like(h)
    dw = np.zeros_like(w)
    peak = 0
    for r0 in range(0, n, rows_per_tile):
        r1 = min(n, r0 + rows_per_tile)
        ht, yt = h[r0:r1], y[r0:r1]
        logits = np.empty((r1 - r0, v))
        peak = max(peak, logits.size)
        lse = np.full(r1 - r0, NEG_INF)
        for c0 in range(0, v, vocab_per_tile):
            blk = mm(ht, w[c0 : c0 + vocab_per_tile].T)
            logits[:, c0 : c0 + blk.shape[1]] = blk
            lse = lse_merge(lse, lse_rows(blk))
        loss[r0:r1] = lse - np.einsum("ij,ij->i", ht, w[yt], optimize=False)
        for c0 in range(0, v, vocab_per_tile):
            blk = logits[:, c0 : c0 + vocab_per_tile]
            np.exp(blk - lse[:, None], out=blk)
            hit = (yt >= c0) & (yt < c0 + blk.shape[1])
            blk[np.nonzero(hit)[0], yt[hit] - c0] -= 1.0
            dh[r0:r1] += mm(blk, w[c0 : c0 + blk.shape[1]])
            dw[c0 : c0 + blk.shape[1]] += mm(blk.T, ht)
    return loss, dh, dw, peak


# ----------------------------------------------------------------- sequence-selective checkpointing


def checkpoint_boundary(split_fraction: float, n: int) -> int:
    """checkpointing.py:48-59: boundary must land on a whole token in (0, N)."""
    exact = split_fraction * n
    b = round(exact)
    if abs(exact - b) > 1e-9 or not 0 < b < n:
        raise ValueError(f"split fraction {split_fraction} does not land on a token boundary for N={n}")
    return int(b)


def checkpoint_plan(policy: str, n: int, d: int, mask: tuple, split_fraction: float | None = None):
    """checkpointing.py:71-97 -> (stored elements, recompute pairs, recompute fraction, extra)."""
    ids = np.arange(1, n + 1)
    am = allowed(mask, ids, ids)
    total = int(am.sum())
    if policy == "full_recompute":
        stored, rec, extra = n * d, total, 0
    elif policy == "selective_pp":
        stored, rec, extra = 2 * n * d, 0, n * d
    else:
        b = checkpoint_boundary(split_fraction, n)
        stored, rec, extra = n * d + (n - b) * d, int(am[:b].sum()), (n - b) * d
    return stored, rec, (rec / total if total else 0.0), extra


def checkpoint_recompute(q, k, v, do, mask: tuple, stored_rows: np.ndarray):
    """checkpointing.py:132-171: keep (O, lse) for stored rows, recompute the rest, backward."""
    n = q.shape[0]
    ids = np.arange(1, n + 1)
    am = allowed(mask, ids, ids)
    o_full, lse_full = attention_forward(q, k, v, am)
    o = np.zeros_like(o_full)
    lse = np.full(n, NEG_INF)
    o[stored_rows] = o_full[stored_rows]
    lse[stored_rows] = lse_full[stored_rows]
    missing = np.setdiff1d(np.arange(n), stored_rows)
    if missing.size:
        s = np.where(am[missing], mm(q[missing], k.T) / math.sqrt(q.shape[1]), NEG_INF)
        lse[missing] = lse_rows(s)
        o[missing] = mm(exp_shifted(s, lse[missing]), v)
    return attention_backward(q, k, v, o, lse, do, am), int(am[missing].sum()) if missing.size else 0
