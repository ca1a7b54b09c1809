"""The callers either side of the ring: burstsim.oracle's layer entry points on
the B200 kernels, and the QKV projection with the layout permutation fused into its GEMM.

* ``AttentionParams`` / ``project_qkv`` (oracle.py:29-44, 60-65): (Q, K, V) = (X Wq, X Wk, X Wv)
  on the tcgen05 GEMM (bf16 operands, fp32 accumulation).
* ``project_qkv_shards``: the same projection for a sharded sequence, where the GEMM's
  store writes token row r straight to its shard-major row (``bb_gemm_bf16_rows`` with the
  inverse of ``shard_token_arrays``' gather) and casts to bf16 — the shards come out of the
  projection in the layout the ring kernels read, with no separate permutation pass over HBM
  (``shard_rows``, distributed.py:104-117, is a gather of the projected matrix).
* ``project_output_shards``: the output projection O W_attn (``AttentionParams.w_attn``) of the
  sharded O, stored in global token order by the same permuting GEMM; the bf16 cast of O is
  fused into the last forward step's merge epilogue (``emit_o_bf16``).
* ``attention_forward`` / ``attention_backward`` (oracle.py:80-119): exact single-device masked
  attention through the ring-step kernels with one device (G = 1).

NumPy inputs give float64 NumPy outputs like the reference; values carry bf16 input rounding
(DESIGN.md §3 tolerances).  CUDA tensors are used in place.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import kernels as K
from .distributed import AttentionGrads, AttentionResult
from .masks import BLOCK_SPARSE, SLIDING_WINDOW, MaskSpec, validate_mask
from .partitioning import ShardLayout, device_token_ids


@dataclass(frozen=True)
class AttentionParams:
    """Square input/output projections of one attention layer (oracle.py:29-44)."""

    dim: int
    w_q: np.ndarray
    w_k: np.ndarray
    w_v: np.ndarray
    w_attn: np.ndarray

    def __post_init__(self):
        for name in ("w_q", "w_k", "w_v", "w_attn"):
            w = getattr(self, name)
            if tuple(w.shape) != (self.dim, self.dim):
                raise ValueError(f"{name} must be {self.dim}x{self.dim}, got {tuple(w.shape)}")


def _device(device) -> torch.device:
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("burst-b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _matrix(x, name: str) -> np.ndarray | torch.Tensor:
    if isinstance(x, torch.Tensor):
        if x.dim() != 2:
            raise ValueError(f"{name} must be a 2-D matrix, got shape {tuple(x.shape)}")
        return x
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"{name} must be a 2-D matrix, got shape {a.shape}")
    return a


def _bf16_padded(x, dev: torch.device, cols: int) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    t = t.to(device=dev, dtype=torch.float32)
    if t.shape[1] < cols:
        t = torch.nn.functional.pad(t, (0, cols - t.shape[1]))
    return t.to(torch.bfloat16).contiguous()


def gemm_rows(x: torch.Tensor, w: torch.Tensor, out: torch.Tensor, row_map: torch.Tensor | None = None) -> None:
    """out[row_map[i]] = bf16(x[i] . w) on the tcgen05 GEMM: x bf16 [m, k], w bf16 [k, n]
    (stored as given, i.e. MN-major B), out bf16 [rows, n]; see bb_gemm_bf16_rows."""
    for t, name in ((x, "x"), (w, "w"), (out, "out")):
        if not t.is_cuda or t.dtype != torch.bfloat16 or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous bf16 CUDA tensor")
    m, k = x.shape
    n = w.shape[1]
    if w.shape[0] != k or out.shape[1] != n:
        raise ValueError(f"gemm_rows: shapes x {tuple(x.shape)}, w {tuple(w.shape)}, out {tuple(out.shape)} disagree")
    if row_map is not None and (row_map.dtype != torch.int64 or not row_map.is_cuda or row_map.shape != (m,)):
        raise ValueError("row_map must be a CUDA int64 vector with one entry per row of x")
    stream = torch.cuda.current_stream(x.device).cuda_stream
    N.check(N.load().bb_gemm_bf16_rows(x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                       None if row_map is None else row_map.data_ptr(), m, n, k, 1, C.c_void_p(stream)))


def _weights(params: AttentionParams, dev: torch.device, kp: int, np_: int) -> list[torch.Tensor]:
    out = []
    for w in (params.w_q, params.w_k, params.w_v):
        t = w if isinstance(w, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(w, dtype=np.float64))
        t = torch.nn.functional.pad(t.to(device=dev, dtype=torch.float32), (0, np_ - t.shape[1], 0, kp - t.shape[0]))
        out.append(t.to(torch.bfloat16).contiguous())
    return out


def project_qkv(x, params: AttentionParams, device=None):
    """(Q, K, V) = (X Wq, X Wk, X Wv) (oracle.py:60-65) on the GPU GEMM."""
    x = _matrix(x, "input embeddings")
    if x.shape[1] != params.dim:
        raise ValueError(f"input has {x.shape[1]} columns, params expect {params.dim}")
    dev = _device(device)
    d = params.dim
    kp = np_ = -(-d // 8) * 8  # TMA rows are 16-byte multiples
    xb = _bf16_padded(x, dev, kp)
    outs = []
    for w in _weights(params, dev, kp, np_):
        o = torch.empty(x.shape[0], np_, dtype=torch.bfloat16, device=dev)
        gemm_rows(xb, w, o)
        outs.append(o[:, :d])
    if isinstance(x, torch.Tensor):
        return tuple(outs)
    return tuple(o.double().cpu().numpy() for o in outs)


def shard_row_map(layout: ShardLayout) -> np.ndarray:
    """int64 [N]: global token row -> its row in the shard-major concatenation of
    ``shard_token_arrays`` (the inverse of the gather ``shard_rows`` performs)."""
    gather = np.concatenate([device_token_ids(layout, i + 1) - 1 for i in range(layout.devices)])
    row_map = np.empty_like(gather)
    row_map[gather] = np.arange(gather.size)
    return row_map.astype(np.int64)


def project_qkv_shards(x, params: AttentionParams, layout: ShardLayout, heads: int = 1, device=None):
    """Projection of the whole sequence straight into per-device shards: returns G tuples
    (Q_i, K_i, V_i) of bf16 [n, heads, dim/heads] CUDA tensors holding the rows of device i in
    shard order (``shard_token_arrays``), written by the GEMM's permuting bf16 store."""
    x = _matrix(x, "input embeddings")
    if x.shape[1] != params.dim:
        raise ValueError(f"input has {x.shape[1]} columns, params expect {params.dim}")
    if x.shape[0] != layout.seq_len:
        raise ValueError(f"input has {x.shape[0]} rows, layout expects {layout.seq_len}")
    if params.dim % heads or (params.dim // heads) % 8:
        raise ValueError(f"dim {params.dim} must split into {heads} heads of a multiple of 8")
    dev = _device(device)
    d, g, n = params.dim, layout.devices, layout.shard_size
    rmap = torch.from_numpy(shard_row_map(layout)).to(dev)
    xb = _bf16_padded(x, dev, d)
    bufs = []
    for w in _weights(params, dev, d, d):
        o = torch.empty(layout.seq_len, d, dtype=torch.bfloat16, device=dev)
        gemm_rows(xb, w, o, rmap)
        bufs.append(o)
    return [tuple(b[i * n:(i + 1) * n].view(n, heads, d // heads) for b in bufs) for i in range(g)]


def _w_attn_padded(params: AttentionParams, heads: int, d_pad: int, cols: int, dev: torch.device) -> torch.Tensor:
    """W_attn as the bf16 [heads * d_pad, cols] B operand of O [n, heads * d_pad]: row h*d_pad + c
    holds W_attn row h*d + c (c < d), padded head columns get zero rows, extra output columns
    (TMA rows are 16-byte multiples) zeros."""
    d = params.dim // heads
    w = params.w_attn if isinstance(params.w_attn, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(params.w_attn, dtype=np.float64))
    w = w.to(device=dev, dtype=torch.float32).view(heads, d, params.dim)
    out = torch.zeros(heads, d_pad, cols, dtype=torch.float32, device=dev)
    out[:, :d, : params.dim] = w
    return out.view(heads * d_pad, cols).to(torch.bfloat16).contiguous()


def project_output_shards(shards, params: AttentionParams, layout: ShardLayout, device=None) -> torch.Tensor:
    """The output projection O W_attn of a sharded sequence (AttentionParams.w_attn,
    oracle.py:29-44), written straight back in global token order.

    ``shards``: the G ``DeviceState``s of a finished ``distributed_forward`` (their bf16 O
    copy when it ran with ``emit_o_bf16=True`` -- the cast fused into the last step's merge
    epilogue -- else their fp32 O, cast by ``bb_cast_pad_bf16``), or G CUDA tensors
    [n, heads, d_pad] (bf16 or fp32) in shard order.  One tcgen05 GEMM per shard whose store
    sends shard row r to global row ``device_token_ids(i)[r] - 1`` (``bb_gemm_bf16_rows``):
    the inverse of shard_rows' gather, with no permutation pass.  Returns bf16 [N, dim]."""
    if len(shards) != layout.devices:
        raise ValueError(f"{len(shards)} shards for a layout of {layout.devices} devices")
    tensors = []
    for s in shards:
        t = getattr(s, "o16", None) if hasattr(s, "o") else s
        if t is None:
            if s.o is None:
                raise RuntimeError("project_output_shards requires a completed forward pass (O missing)")
            t = s.o
        tensors.append(t)
    dev = _device(device) if device is not None else tensors[0].device
    n, heads, d_pad = tensors[0].shape
    if params.dim % heads:
        raise ValueError(f"dim {params.dim} does not split into {heads} heads")
    if params.dim // heads > d_pad:
        raise ValueError(f"shards hold {d_pad} columns per head, params need {params.dim // heads}")
    cols = -(-params.dim // 8) * 8
    for i, t in enumerate(tensors):
        if t.shape != (layout.shard_size, heads, d_pad):
            raise ValueError(f"shard {i + 1} has shape {tuple(t.shape)}, expected ({layout.shard_size}, {heads}, {d_pad})")
    with torch.cuda.device(dev):
        w = _w_attn_padded(params, heads, d_pad, cols, dev)
        out = torch.empty(layout.seq_len, cols, dtype=torch.bfloat16, device=dev)
        for i, t in enumerate(tensors):
            t = t.to(dev)
            if t.dtype == torch.float32:
                t = K.cast_pad_bf16(t.contiguous(), d_pad)
            rows = torch.from_numpy(device_token_ids(layout, i + 1) - 1).to(dev)
            gemm_rows(t.contiguous().view(n, heads * d_pad), w, out, rows)
    return out[:, : params.dim]


def _first_empty_row(mask: MaskSpec, nq: int, nk: int) -> int | None:
    """0-based first query row with no allowed key among keys 1..nk (oracle.py:88-91 raises
    for it).  Full and causal masks always leave key 1; a sliding window empties rows
    q >= nk + w; a block-sparse mask empties rows whose block row has no block before nk."""
    if mask.kind == SLIDING_WINDOW:
        r = nk + int(mask.window) - 1  # first id q = r + 1 with q - nk >= w
        return r if r < nq else None
    if mask.kind != BLOCK_SPARSE:
        return None
    bm = np.asarray(mask.block_mask) != 0
    bl = int(mask.block_len)
    for r in range(nq):
        blk = bm[r // bl, : -(-nk // bl)]
        if not blk.any():
            return r
    return None


def masked_scores(q, k, mask: MaskSpec, device=None):
    """S = Q K^T / sqrt(d) with masked-out entries -inf (oracle.py:66-75), float64 on the device:
    the fp64 GEMM with K^T as a stride swap, then one pass that scales and applies the
    reference's dense allowed-pair matrix (``dense_mask``, host logic as in the reference)."""
    from . import numerics as F
    from .masks import dense_mask

    dev = q.device if isinstance(q, torch.Tensor) and q.is_cuda else _device(device)
    host = not (isinstance(q, torch.Tensor) and q.is_cuda)
    qt, kt = F._as(q, 2, "Q", dev), F._as(k, 2, "K", dev)
    if qt.shape[1] != kt.shape[1]:
        raise ValueError(f"Q has dim {qt.shape[1]} but K has dim {kt.shape[1]}")
    validate_mask(mask, max(qt.shape[0], kt.shape[0]))
    s = F.matmul(qt, kt.t())
    allowed = torch.from_numpy(np.ascontiguousarray(dense_mask(mask, qt.shape[0], kt.shape[0]), dtype=np.uint8)).to(dev)
    with torch.cuda.device(dev):
        N.check(N.load().bb_scale_mask_f64(s.data_ptr(), allowed.data_ptr(), math.sqrt(qt.shape[1]), s.numel(),
                                           C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return s.cpu().numpy() if host else s


def _single_device_layout(nq: int, nk: int) -> ShardLayout:
    """One shard holding ids 1..max(nq, nk): queries are its first nq rows, keys its first nk
    (dense_mask's id convention, masks.py:89-104); rows past either count are never read."""
    return ShardLayout("contiguous", max(nq, nk), 1)


def attention_forward(q, k, v, mask: MaskSpec, device=None) -> AttentionResult:
    """O = softmax(Q K^T / sqrt(d)) V and the row LSE (oracle.py:80-95), one device."""
    q, k, v = _matrix(q, "Q"), _matrix(k, "K"), _matrix(v, "V")
    if k.shape[0] != v.shape[0]:
        raise ValueError(f"K has {k.shape[0]} rows but V has {v.shape[0]}")
    if q.shape[1] != k.shape[1] or k.shape[1] != v.shape[1]:
        raise ValueError("Q, K, V must share the model dimension")
    nq, nk, d = q.shape[0], k.shape[0], q.shape[1]
    validate_mask(mask, max(nq, nk))
    bad = _first_empty_row(mask, nq, nk)
    if bad is not None:
        raise ValueError(f"query row {bad + 1} has no unmasked key")
    dev = _device(device)
    dp = 64 if d <= 64 else 128
    if d > 128:
        raise ValueError(f"model dimension {d} > 128: split it into heads (the kernels take d <= 128)")
    with torch.cuda.device(dev):
        qb, kb, vb = (_bf16_padded(t, dev, dp).view(-1, 1, dp) for t in (q, k, v))
        o = torch.zeros(nq, 1, dp, device=dev)
        lse = torch.full((1, nq), float("-inf"), device=dev)
        K.attn_fwd_step(qb, kb, vb, o, lse, _single_device_layout(nq, nk), K.device_mask(mask, dev), 1, 1,
                        1.0 / math.sqrt(d), n_q=nq)
    res = AttentionResult(o=o[:, 0, :d], lse=lse[0])
    if isinstance(q, torch.Tensor):
        return res
    return AttentionResult(o=res.o.double().cpu().numpy(), lse=res.lse.double().cpu().numpy())


def attention_backward(q, k, v, o, lse, do, mask: MaskSpec, device=None) -> AttentionGrads:
    """Gradients of sum(O * dO) w.r.t. Q, K, V (oracle.py:98-119), one device.

    Checks what the reference's masked_scores / matmul chain rejects (oracle.py:66-75,
    108-119) before any device memory is touched: Q/K model dims, K/V rows, dO and O shapes,
    the mask against max(nq, nk), and the lse length."""
    q, k, v, do = _matrix(q, "Q"), _matrix(k, "K"), _matrix(v, "V"), _matrix(do, "dO")
    o = _matrix(o, "O")
    if tuple(do.shape) != (q.shape[0], v.shape[1]):
        raise ValueError(f"dO must be {q.shape[0]}x{v.shape[1]}, got {tuple(do.shape)}")
    if q.shape[1] != k.shape[1]:
        raise ValueError(f"Q has dim {q.shape[1]} but K has dim {k.shape[1]}")
    if k.shape[0] != v.shape[0]:
        raise ValueError(f"K has {k.shape[0]} rows but V has {v.shape[0]}")
    if v.shape[1] != q.shape[1]:
        raise ValueError("Q, K, V must share the model dimension")
    if tuple(o.shape) != tuple(do.shape):
        raise ValueError(f"O must be {do.shape[0]}x{do.shape[1]}, got {tuple(o.shape)}")
    nq, nk, d = q.shape[0], k.shape[0], q.shape[1]
    validate_mask(mask, max(nq, nk))
    lt = lse if isinstance(lse, torch.Tensor) else torch.from_numpy(np.asarray(lse, dtype=np.float64))
    if lt.numel() != nq:
        raise ValueError(f"lse must have {nq} entries, got {lt.numel()}")
    if d > 128:
        raise ValueError(f"model dimension {d} > 128: split it into heads (the kernels take d <= 128)")
    dev = _device(device)
    dp = 64 if d <= 64 else 128
    with torch.cuda.device(dev):
        qb, kb, vb, dob = (_bf16_padded(t, dev, dp).view(-1, 1, dp) for t in (q, k, v, do))
        ot = o if isinstance(o, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(o))
        ot = torch.nn.functional.pad(ot.to(device=dev, dtype=torch.float32), (0, dp - d)).view(-1, 1, dp).contiguous()
        lt = lt.to(device=dev, dtype=torch.float32).reshape(1, nq).contiguous()
        delta = torch.empty(1, nq, device=dev)
        K.bwd_preprocess(dob, ot, delta)
        dq = torch.zeros(nq, 1, dp, device=dev)
        dk = torch.zeros(nk, 1, dp, device=dev)
        dv = torch.zeros(nk, 1, dp, device=dev)
        K.attn_bwd_step(qb, kb, vb, dob, lt, delta, dq, dk, dv, _single_device_layout(nq, nk), K.device_mask(mask, dev),
                        1, 1, 1.0 / math.sqrt(d))
    grads = AttentionGrads(dq=dq[:, 0, :d], dk=dk[:, 0, :d], dv=dv[:, 0, :d])
    if isinstance(q, torch.Tensor):
        return grads
    return AttentionGrads(*(t.double().cpu().numpy() for t in (grads.dq, grads.dk, grads.dv)))


@dataclass(frozen=True)
class LmHeadResult:
    """oracle.py:121-126: per-token loss (nats), dH, dW."""

    loss: np.ndarray
    dh: np.ndarray
    dw: np.ndarray


def naive_lmhead_loss(h, w_head, targets, device=None) -> LmHeadResult:
    """Full-materialisation LM head + cross entropy with analytic gradients (oracle.py:129-154).

    Float64 end to end on the device (``numerics`` kernels): logits = H W^T, row LSE,
    loss = lse - logit[y], dlogits = softmax - onehot(y) in one pass, dH = G W, dW = G^T H
    (the transposes are stride swaps).  This is the float64 check of the bf16 fused head
    (``fused_lmhead_loss``); NumPy inputs give NumPy outputs.
    """
    from . import numerics as F

    dev = h.device if isinstance(h, torch.Tensor) and h.is_cuda else _device(device)
    host = not (isinstance(h, torch.Tensor) and h.is_cuda)
    ht = F._as(h, 2, "H", dev)
    wt = F._as(w_head, 2, "W_head", dev)
    y = targets.detach().to("cpu") if isinstance(targets, torch.Tensor) else targets
    y = np.asarray(y, dtype=np.int64)
    n, d = ht.shape
    v = wt.shape[0]
    if wt.shape[1] != d:
        raise ValueError(f"W_head must have {d} columns, got {wt.shape[1]}")
    if y.shape != (n,):
        raise ValueError(f"targets must have length {n}, got shape {y.shape}")
    bad = np.nonzero((y < 0) | (y >= v))[0]
    if bad.size:
        raise ValueError(f"target index {y[bad[0]]} at row {int(bad[0])} outside [0, {v})")
    yt = torch.from_numpy(y).to(dev)
    logits = F.matmul(ht, wt.t())
    lse = F.row_logsumexp(logits) if n else torch.empty(0, dtype=torch.float64, device=dev)
    loss, g = F.softmax_xent(logits, lse, yt)
    dh = F.matmul(g, wt)
    dw = F.matmul(g.t(), ht)
    if host:
        return LmHeadResult(loss=loss.cpu().numpy(), dh=dh.cpu().numpy(), dw=dw.cpu().numpy())
    return LmHeadResult(loss=loss, dh=dh, dw=dw)


def finite_diff_check(f, x, analytic_grad, h: float = 1e-6) -> float:
    """oracle.py:157-187: worst relative error of central differences of ``f`` against
    ``analytic_grad`` (denominator max(|analytic|, 1e-8) per entry).  Host-side test
    utility: ``f`` is the caller's function and runs wherever it runs."""
    from .numerics import as_matrix

    if h <= 0:
        raise ValueError(f"step size must be positive, got {h}")
    x = as_matrix(x, "finite-difference point")
    g = as_matrix(analytic_grad, "analytic gradient")
    if g.shape != x.shape:
        raise ValueError(f"gradient shape {g.shape} != point shape {x.shape}")
    worst = 0.0
    probe = x.copy()
    for idx in np.ndindex(*x.shape):
        centre = x[idx]
        probe[idx] = centre + h
        hi = float(f(probe.copy()))
        probe[idx] = centre - h
        lo = float(f(probe.copy()))
        probe[idx] = centre
        if not (math.isfinite(hi) and math.isfinite(lo)):
            raise ValueError(f"f is non-finite near entry {idx}")
        err = abs((hi - lo) / (2.0 * h) - g[idx]) / max(abs(g[idx]), 1e-8)
        worst = max(worst, float(err))
    return worst
