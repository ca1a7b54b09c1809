"""torch-tensor front end of the C ABI: one function per exported kernel.

Tensors are plumbing here (device memory + streams); every call goes straight
to libburst_b200.so on the tensor's device and current torch stream.  There is
no CPU path: a CPU tensor, a wrong dtype or a missing library raises.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
import struct
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .masks import BLOCK_SPARSE, SLIDING_WINDOW, MaskSpec
from .partitioning import ShardLayout


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _require(t: torch.Tensor, dtype: torch.dtype, name: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback), got {t.device}")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def layout_struct(layout: ShardLayout) -> N.BbLayout:
    return N.BbLayout(
        kind=N.LAYOUT_CODES[layout.kind],
        devices=layout.devices,
        seq_len=layout.seq_len,
        block_len=int(layout.block_len or 0),
    )


@dataclass
class DeviceMask:
    """MaskSpec lowered for the kernels on one device (block mask as uint8 in HBM)."""

    spec: MaskSpec
    struct: N.BbMask
    block_mask: torch.Tensor | None  # keeps the device copies alive
    spans: torch.Tensor | None = None


_MASK_CACHE_SIZE = 16
_mask_cache: "OrderedDict[tuple, DeviceMask]" = OrderedDict()


def _mask_key(mask: MaskSpec, dev_index: int) -> tuple:
    """Content key: a MaskSpec edited in place, or a new one with equal contents, maps to the
    device copy of exactly those contents (never a stale one)."""
    bm = None
    if mask.kind == BLOCK_SPARSE and mask.block_mask is not None:
        a = np.ascontiguousarray(np.asarray(mask.block_mask) != 0)
        bm = (a.shape, hashlib.blake2b(a.tobytes(), digest_size=16).digest())
    return (mask.kind, mask.window, mask.block_len, bm, dev_index)


def device_mask(mask: MaskSpec, device: torch.device) -> DeviceMask:
    key = _mask_key(mask, device.index if device.index is not None else torch.cuda.current_device())
    hit = _mask_cache.get(key)
    if hit is not None:
        _mask_cache.move_to_end(key)
        return hit
    bm = spans = None
    s = N.BbMask(kind=N.MASK_CODES[mask.kind], reserved=0, window=0, block_len=0, num_blocks=0, block_mask=None)
    if mask.kind == SLIDING_WINDOW:
        s.window = int(mask.window)
    if mask.kind == BLOCK_SPARSE:
        m = np.asarray(mask.block_mask) != 0
        bm = torch.from_numpy(np.ascontiguousarray(m, dtype=np.uint8)).to(device)
        s.block_len = int(mask.block_len)
        s.num_blocks = int(m.shape[0])
        s.block_mask = bm.data_ptr()
        spans = torch.from_numpy(np.concatenate([_spans(m), _spans(m.T)])).to(device)
        s.row_span = spans.data_ptr()
        s.col_span = spans.data_ptr() + m.shape[0] * 2 * 4
    dm = DeviceMask(mask, s, bm, spans)
    _mask_cache[key] = dm
    while len(_mask_cache) > _MASK_CACHE_SIZE:  # bounded: device copies of old masks are released
        _mask_cache.popitem(last=False)
    return dm


def _spans(m: np.ndarray) -> np.ndarray:
    """[rows, 2] int32: first and last nonzero column per row of a 0/1 block mask, -1 if none."""
    any_ = m.any(axis=1)
    first = np.where(any_, m.argmax(axis=1), -1)
    last = np.where(any_, m.shape[1] - 1 - m[:, ::-1].argmax(axis=1), -1)
    return np.ascontiguousarray(np.stack([first, last], axis=1), dtype=np.int32)


def attn_fwd_step(
    q: torch.Tensor,
    k: torch.Tensor,
    v: torch.Tensor,
    o: torch.Tensor,
    lse: torch.Tensor,
    layout: ShardLayout,
    mask: DeviceMask,
    q_device: int,
    k_device: int,
    softmax_scale: float,
    n_q: int | None = None,
    o_bf16: torch.Tensor | None = None,
) -> None:
    """Fold key shard ``k_device`` into device ``q_device``'s running (O, lse); see bb_attn_fwd_step.
    ``o_bf16`` (bf16, O's shape): also store bf16(O) of every row after the merge (last step)."""
    for t, name in ((q, "Q"), (k, "K"), (v, "V")):
        _require(t, torch.bfloat16, name)
    _require(o, torch.float32, "O")
    _require(lse, torch.float32, "lse")
    if o_bf16 is not None:
        _require(o_bf16, torch.bfloat16, "O (bf16 copy)")
        if o_bf16.shape != o.shape:
            raise ValueError(f"bf16 O copy has shape {tuple(o_bf16.shape)}, O has {tuple(o.shape)}")
    nq = q.shape[0] if n_q is None else n_q
    a = N.BbAttnFwdArgs(
        q=_ptr(q), k=_ptr(k), v=_ptr(v), o=_ptr(o), lse=_ptr(lse),
        n_q=nq, n_k=k.shape[0], hq=q.shape[1], hkv=k.shape[1], head_dim=q.shape[2],
        softmax_scale=float(softmax_scale), q_device=q_device, k_device=k_device,
        layout=layout_struct(layout), mask=mask.struct, o_bf16=_ptr(o_bf16) if o_bf16 is not None else None,
    )
    N.check(N.load().bb_attn_fwd_step(C.byref(a), C.c_void_p(_stream(q.device))))


def attn_bwd_step(
    q, k, v, dout, lse, delta, dq, dk, dv,
    layout: ShardLayout, mask: DeviceMask, q_device: int, k_device: int, softmax_scale: float,
    kv_heads: tuple[int, int] | None = None,
) -> None:
    """Accumulate one (query shard, key shard) pair into dq/dk/dv; see bb_attn_bwd_step.
    ``kv_heads=(b, e)`` restricts the step to kv heads [b, e) and their query heads."""
    for t, name in ((q, "Q"), (k, "K"), (v, "V"), (dout, "dO")):
        _require(t, torch.bfloat16, name)
    for t, name in ((lse, "lse"), (delta, "D"), (dq, "dQ"), (dk, "dK"), (dv, "dV")):
        _require(t, torch.float32, name)
    a = N.BbAttnBwdArgs(
        q=_ptr(q), k=_ptr(k), v=_ptr(v), dout=_ptr(dout), lse=_ptr(lse), delta=_ptr(delta),
        dq=_ptr(dq), dk=_ptr(dk), dv=_ptr(dv),
        n_q=q.shape[0], n_k=k.shape[0], hq=q.shape[1], hkv=k.shape[1], head_dim=q.shape[2],
        softmax_scale=float(softmax_scale), q_device=q_device, k_device=k_device,
        layout=layout_struct(layout), mask=mask.struct,
        kv_head_begin=kv_heads[0] if kv_heads else 0, kv_head_end=kv_heads[1] if kv_heads else 0,
    )
    N.check(N.load().bb_attn_bwd_step(C.byref(a), C.c_void_p(_stream(q.device))))


def bwd_preprocess(dout: torch.Tensor, o: torch.Tensor, delta: torch.Tensor) -> None:
    """delta[h, r] = rowsum(dO o O) (distributed.py:274-275)."""
    _require(dout, torch.bfloat16, "dO")
    _require(o, torch.float32, "O")
    _require(delta, torch.float32, "D")
    n, h, d = dout.shape
    N.check(N.load().bb_attn_bwd_preprocess(_ptr(dout), _ptr(o), _ptr(delta), n, h, d, C.c_void_p(_stream(o.device))))


def permute_rows(dst: torch.Tensor, src: torch.Tensor, index: torch.Tensor, scatter: bool) -> None:
    """gather: dst[r] = src[index[r]]; scatter: dst[index[r]] = src[r] (0-based rows)."""
    if not (dst.is_cuda and src.is_cuda and index.is_cuda):
        raise ValueError("permute_rows needs CUDA tensors")
    if index.dtype != torch.int64:
        raise ValueError("permute_rows index must be int64")
    rows = index.shape[0]
    row_bytes = src[0].numel() * src.element_size() if src.shape[0] else 0
    N.check(
        N.load().bb_permute_rows(_ptr(dst), _ptr(src), _ptr(index), rows, row_bytes, int(scatter), C.c_void_p(_stream(src.device)))
    )


def set_split_rows(rows: int = 0) -> None:
    """Test hook (bb_debug_set_split_rows): shard size above which one ring-step call is
    launched as sub-shard pairs; 0 restores the default (the kernels' 524288-row tables)."""
    N.check(N.load().bb_debug_set_split_rows(int(rows)))


def fill_(t: torch.Tensor, value: float = 0.0) -> torch.Tensor:
    """In-place fill of a contiguous fp32 tensor (bb_fill_u32); returns ``t``."""
    _require(t, torch.float32, "fill target")
    bits = struct.unpack("<I", struct.pack("<f", value))[0]
    with torch.cuda.device(t.device):
        N.check(N.load().bb_fill_u32(_ptr(t), bits, t.numel(), C.c_void_p(_stream(t.device))))
    return t


def _row_view(t: torch.Tensor, name: str) -> tuple[int, int, int]:
    """(rows, cols, row stride) of a tensor whose rows are contiguous runs (t[r] dense)."""
    inner = 1
    for size, stride in zip(reversed(t.shape[1:]), reversed(t.stride()[1:])):
        if size != 1 and stride != inner:
            raise ValueError(f"{name}: every row must be one contiguous run")
        inner *= size
    return t.shape[0], inner, t.stride(0) if t.dim() > 1 else inner


def add_rows_(dst: torch.Tensor, src: torch.Tensor) -> torch.Tensor:
    """dst += src for fp32 tensors of one shape whose rows are contiguous runs (a whole
    accumulator or a head range ``x[:, a:b]`` of one), on bb_add_rows_f32; returns ``dst``."""
    _require_cuda_f32(dst, "fold target")
    _require_cuda_f32(src, "fold source")
    if dst.shape != src.shape:
        raise ValueError(f"fold shapes differ: {tuple(dst.shape)} vs {tuple(src.shape)}")
    rows, cols, dld = _row_view(dst, "fold target")
    _, _, sld = _row_view(src, "fold source")
    with torch.cuda.device(dst.device):
        N.check(N.load().bb_add_rows_f32(_ptr(dst), _ptr(src), rows, cols, dld, sld, C.c_void_p(_stream(dst.device))))
    return dst


def _require_cuda_f32(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback), got {t.device}")
    if t.dtype != torch.float32:
        raise ValueError(f"{name} must be torch.float32, got {t.dtype}")


def cast_pad_bf16(src: torch.Tensor, cols_out: int) -> torch.Tensor:
    """f32 [..., c] -> bf16 [..., cols_out] with zero padding (cols_out >= c)."""
    _require(src, torch.float32, "src")
    cin = src.shape[-1]
    rows = src.numel() // max(cin, 1)
    out = torch.empty(*src.shape[:-1], cols_out, dtype=torch.bfloat16, device=src.device)
    with torch.cuda.device(src.device):
        N.check(N.load().bb_cast_pad_bf16(_ptr(out), _ptr(src), rows, cin, cols_out, C.c_void_p(_stream(src.device))))
    return out


def gemm(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor, m: int, n: int, k: int, a_mn: bool, b_mn: bool, accumulate: bool) -> None:
    _require(a, torch.bfloat16, "A")
    _require(b, torch.bfloat16, "B")
    _require(c, torch.float32, "C")
    N.check(
        N.load().bb_gemm_bf16(_ptr(a), _ptr(b), _ptr(c), m, n, k, int(a_mn), int(b_mn), int(accumulate), C.c_void_p(_stream(a.device)))
    )


def lmhead_workspace_bytes(n: int, vocab: int, dim: int, rows_per_tile: int) -> int:
    return int(N.load().bb_lmhead_workspace_bytes(n, vocab, dim, rows_per_tile))


def lmhead_fused(
    h: torch.Tensor, w: torch.Tensor, targets: torch.Tensor, loss: torch.Tensor, dh: torch.Tensor,
    dw: torch.Tensor, rows_per_tile: int, vocab_per_tile: int, workspace: torch.Tensor,
) -> None:
    _require(h, torch.bfloat16, "H")
    _require(w, torch.bfloat16, "W_head")
    if targets.dtype != torch.int64 or not targets.is_cuda:
        raise ValueError("targets must be a CUDA int64 tensor")
    for t, name in ((loss, "loss"), (dh, "dH"), (dw, "dW")):
        _require(t, torch.float32, name)
    a = N.BbLmheadArgs(
        h=_ptr(h), w=_ptr(w), targets=_ptr(targets), n=h.shape[0], vocab=w.shape[0], dim=h.shape[1],
        rows_per_tile=int(rows_per_tile), vocab_per_tile=int(vocab_per_tile),
        loss=_ptr(loss), dh=_ptr(dh), dw=_ptr(dw), workspace=_ptr(workspace), workspace_bytes=workspace.numel(),
    )
    N.check(N.load().bb_lmhead_fused(C.byref(a), C.c_void_p(_stream(h.device))))


def debug_mask_tiles(layout: ShardLayout, mask: DeviceMask, q_device: int, k_device: int, n_q: int, n_k: int,
                     view: str, device: torch.device) -> tuple[np.ndarray, np.ndarray]:
    """The tile classes ([n_q/128, n_k/128] int8: 0 skip, 1 full, 2 partial) and the element
    mask ([n_q, n_k] bool) that the forward (``view="fwd"``) or backward (``"bwd"``) kernel
    realises for ring step (q_device, k_device); see bb_debug_mask_tiles."""
    n_qt, n_kt = -(-n_q // 128), -(-n_k // 128)
    cls = torch.zeros(n_qt * n_kt, dtype=torch.int8, device=device)
    allowed = torch.zeros(n_q * n_k, dtype=torch.uint8, device=device)
    lay = layout_struct(layout)
    with torch.cuda.device(device):
        N.check(N.load().bb_debug_mask_tiles(C.byref(lay), C.byref(mask.struct), q_device, k_device, n_q, n_k,
                                             {"fwd": 0, "bwd": 1}[view], _ptr(cls), _ptr(allowed),
                                             C.c_void_p(_stream(device))))
    return cls.cpu().numpy().reshape(n_qt, n_kt), allowed.cpu().numpy().reshape(n_q, n_k).astype(bool)


def padded_head_dim(d: int) -> int:
    """Head dims the kernels take: 64 or 128 (smaller dims are zero-padded, scale unchanged)."""
    if d <= 64:
        return 64
    if d <= 128:
        return 128
    raise ValueError(f"head_dim {d} > 128 is not supported by the sm_100a kernels")


def default_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)
