"""ctypes binding of the C ABI in include/burst_b200.h (libburst_b200.so).

This is the only module that touches the shared library.  There is no
fallback: if the library is missing or a call fails, an exception is raised
(ValueError for BB_ERR_INVALID, RuntimeError otherwise), mirroring the
reference's error types (SURVEY.md §8b "Errors").
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("BB_LIB_PATH") or Path(__file__).resolve().parent / "_lib" / "libburst_b200.so")

BB_OK, BB_ERR_INVALID, BB_ERR_CUDA, BB_ERR_UNSUPPORTED = 0, 1, 2, 3

LAYOUT_CODES = {"contiguous": 0, "zigzag": 1, "striped": 2, "block_striped": 3}
MASK_CODES = {"full": 0, "causal": 1, "sliding_window": 2, "block_sparse": 3}

# Every symbol include/burst_b200.h declares (checked by the CPU test suite).
EXPORTS = (
    "bb_attn_fwd_step",
    "bb_attn_bwd_step",
    "bb_attn_bwd_preprocess",
    "bb_permute_rows",
    "bb_cast_pad_bf16",
    "bb_fill_u32",
    "bb_debug_set_split_rows",
    "bb_add_rows_f32",
    "bb_lmhead_workspace_bytes",
    "bb_lmhead_fused",
    "bb_gemm_bf16",
    "bb_gemm_bf16_rows",
    "bb_ipc_handle_bytes",
    "bb_arena_alloc",
    "bb_arena_free",
    "bb_ipc_export",
    "bb_ipc_import",
    "bb_ipc_close",
    "bb_copy_async",
    "bb_flag_write",
    "bb_flag_wait",
    "bb_matmul_f64",
    "bb_scale_mask_f64",
    "bb_row_logsumexp_f64",
    "bb_lse_merge_f64",
    "bb_exp_shifted_f64",
    "bb_exp_gap_f64",
    "bb_rowsum_hadamard_f64",
    "bb_xent_f64",
    "bb_last_error",
    "bb_debug_probe",
    "bb_debug_mask_tiles",
    "bb_abi_version",
    "bb_launch_count",
)


class BbLayout(C.Structure):
    _fields_ = [("kind", C.c_int32), ("devices", C.c_int32), ("seq_len", C.c_int64), ("block_len", C.c_int64)]


class BbMask(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("reserved", C.c_int32),
        ("window", C.c_int64),
        ("block_len", C.c_int64),
        ("num_blocks", C.c_int64),
        ("block_mask", C.c_void_p),
        ("row_span", C.c_void_p),
        ("col_span", C.c_void_p),
    ]


class BbAttnFwdArgs(C.Structure):
    _fields_ = [
        ("q", C.c_void_p),
        ("k", C.c_void_p),
        ("v", C.c_void_p),
        ("o", C.c_void_p),
        ("lse", C.c_void_p),
        ("n_q", C.c_int64),
        ("n_k", C.c_int64),
        ("hq", C.c_int32),
        ("hkv", C.c_int32),
        ("head_dim", C.c_int32),
        ("softmax_scale", C.c_float),
        ("q_device", C.c_int32),
        ("k_device", C.c_int32),
        ("layout", BbLayout),
        ("mask", BbMask),
        ("o_bf16", C.c_void_p),
    ]


class BbAttnBwdArgs(C.Structure):
    _fields_ = [
        ("q", C.c_void_p),
        ("k", C.c_void_p),
        ("v", C.c_void_p),
        ("dout", C.c_void_p),
        ("lse", C.c_void_p),
        ("delta", C.c_void_p),
        ("dq", C.c_void_p),
        ("dk", C.c_void_p),
        ("dv", C.c_void_p),
        ("n_q", C.c_int64),
        ("n_k", C.c_int64),
        ("hq", C.c_int32),
        ("hkv", C.c_int32),
        ("head_dim", C.c_int32),
        ("softmax_scale", C.c_float),
        ("q_device", C.c_int32),
        ("k_device", C.c_int32),
        ("layout", BbLayout),
        ("mask", BbMask),
        ("kv_head_begin", C.c_int32),
        ("kv_head_end", C.c_int32),
    ]


class BbLmheadArgs(C.Structure):
    _fields_ = [
        ("h", C.c_void_p),
        ("w", C.c_void_p),
        ("targets", C.c_void_p),
        ("n", C.c_int64),
        ("vocab", C.c_int64),
        ("dim", C.c_int64),
        ("rows_per_tile", C.c_int64),
        ("vocab_per_tile", C.c_int64),
        ("loss", C.c_void_p),
        ("dh", C.c_void_p),
        ("dw", C.c_void_p),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_int64),
    ]


_lib: C.CDLL | None = None


def load(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"burst-b200 kernel library not built: {p} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`)"
        )
    lib = C.CDLL(str(p))
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    lib.bb_attn_fwd_step.argtypes = [C.POINTER(BbAttnFwdArgs), vp]
    lib.bb_attn_bwd_step.argtypes = [C.POINTER(BbAttnBwdArgs), vp]
    lib.bb_attn_bwd_preprocess.argtypes = [vp, vp, vp, i64, i32, i32, vp]
    lib.bb_permute_rows.argtypes = [vp, vp, vp, i64, i64, i32, vp]
    lib.bb_cast_pad_bf16.argtypes = [vp, vp, i64, i32, i32, vp]
    lib.bb_fill_u32.argtypes = [vp, C.c_uint32, i64, vp]
    lib.bb_debug_set_split_rows.argtypes = [i64]
    lib.bb_add_rows_f32.argtypes = [vp, vp, i64, i64, i64, i64, vp]
    lib.bb_lmhead_workspace_bytes.argtypes = [i64, i64, i64, i64]
    lib.bb_lmhead_workspace_bytes.restype = i64
    lib.bb_lmhead_fused.argtypes = [C.POINTER(BbLmheadArgs), vp]
    lib.bb_gemm_bf16.argtypes = [vp, vp, vp, i64, i64, i64, i32, i32, i32, vp]
    lib.bb_gemm_bf16_rows.argtypes = [vp, vp, vp, vp, i64, i64, i64, i32, vp]
    lib.bb_ipc_handle_bytes.restype = i32
    lib.bb_arena_alloc.argtypes = [i64, C.POINTER(vp)]
    lib.bb_arena_free.argtypes = [vp]
    lib.bb_ipc_export.argtypes = [vp, vp]
    lib.bb_ipc_import.argtypes = [vp, C.POINTER(vp)]
    lib.bb_ipc_close.argtypes = [vp]
    lib.bb_copy_async.argtypes = [vp, vp, i64, vp]
    lib.bb_flag_write.argtypes = [vp, C.c_uint32, vp]
    lib.bb_flag_wait.argtypes = [vp, C.c_uint32, vp]
    lib.bb_matmul_f64.argtypes = [vp, i64, i64, vp, i64, i64, vp, i64, i64, i64, vp]
    lib.bb_scale_mask_f64.argtypes = [vp, vp, C.c_double, i64, vp]
    lib.bb_row_logsumexp_f64.argtypes = [vp, i64, i64, i64, vp, vp]
    lib.bb_lse_merge_f64.argtypes = [vp, vp, vp, i64, vp]
    lib.bb_exp_shifted_f64.argtypes = [vp, vp, vp, i64, i64, vp]
    lib.bb_exp_gap_f64.argtypes = [vp, vp, vp, i64, vp]
    lib.bb_rowsum_hadamard_f64.argtypes = [vp, vp, vp, i64, i64, vp]
    lib.bb_xent_f64.argtypes = [vp, vp, vp, i64, i64, vp, vp, vp]
    lib.bb_last_error.restype = C.c_char_p
    lib.bb_debug_probe.argtypes = [vp, i32]
    lib.bb_debug_mask_tiles.argtypes = [C.POINTER(BbLayout), C.POINTER(BbMask), i32, i32, i64, i64, i32, vp, vp, vp]
    lib.bb_abi_version.restype = i32
    lib.bb_launch_count.restype = i64
    for name in EXPORTS:
        if name not in ("bb_lmhead_workspace_bytes", "bb_ipc_handle_bytes", "bb_last_error", "bb_abi_version", "bb_launch_count"):
            getattr(lib, name).restype = C.c_int
    if path is None:
        _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == BB_OK:
        return
    msg = load().bb_last_error().decode(errors="replace")
    if rc == BB_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"burst-b200 error {rc}: {msg}")


def launch_count() -> int:
    return int(load().bb_launch_count())
