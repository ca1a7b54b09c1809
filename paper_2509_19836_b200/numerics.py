"""Float64 tile math -- drop-in for burstsim.numerics (numerics.py:1-116) on the B200.

Same names, argument meaning and errors as the reference; the arithmetic runs in
the float64 kernels of ``csrc/bb_numerics.cu`` (C ABI ``bb_*_f64``).  ``-inf`` stays
an exact "no mass" sentinel (``lse_merge(-inf, x) == x``, ``exp_gap(-inf, .) == 0``,
numerics.py:62-69,101-116) and every reduction has a fixed order, so results are
bit-identical run to run (numerics.py:1-11).

Arguments may be NumPy arrays / nested lists (the reference's inputs: copied to
the current CUDA device, the result comes back as ``np.ndarray``) or float64 CUDA
tensors (kept on their device, the result is a tensor there).  There is no CPU
path: without the kernel library or a GPU the call raises.
``seeded_random_matrix`` is the reference's input generator (PCG64, U[-1, 1],
numerics.py:95-98); it stays on the host so seeds give the reference's values.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N

NEG_INF = float("-inf")


def _dev_of(*xs) -> torch.device:
    for x in xs:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return x.device
    if not torch.cuda.is_available():
        raise RuntimeError("burst-b200 numerics need a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _host_out(*xs) -> bool:
    return not any(isinstance(x, torch.Tensor) and x.is_cuda for x in xs)


def _as(x, ndim: int, name: str, dev: torch.device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.detach()
    else:
        t = torch.from_numpy(np.asarray(x, dtype=np.float64))
    if t.ndim != ndim:
        kind = "2-dimensional" if ndim == 2 else "1-dimensional"
        raise ValueError(f"{name} must be {kind}, got shape {tuple(t.shape)}")
    return t.to(device=dev, dtype=torch.float64)


def as_matrix(a, name: str = "matrix") -> np.ndarray:
    """numerics.py:21-25 (host-side coercion, used for argument checking)."""
    out = np.asarray(a, dtype=np.float64)
    if out.ndim != 2:
        raise ValueError(f"{name} must be 2-dimensional, got shape {out.shape}")
    return out


def as_vector(a, name: str = "vector") -> np.ndarray:
    """numerics.py:28-32."""
    out = np.asarray(a, dtype=np.float64)
    if out.ndim != 1:
        raise ValueError(f"{name} must be 1-dimensional, got shape {out.shape}")
    return out


def _stream(dev: torch.device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _ret(t: torch.Tensor, host: bool):
    return t.cpu().numpy() if host else t


def matmul(a, b):
    """numerics.py:35-45: a @ b in float64, k accumulated in ascending order."""
    dev, host = _dev_of(a, b), _host_out(a, b)
    ta, tb = _as(a, 2, "matmul operand a", dev), _as(b, 2, "matmul operand b", dev)
    if ta.shape[1] != tb.shape[0]:
        raise ValueError(
            f"matmul shape mismatch: a is {ta.shape[0]}x{ta.shape[1]}, b is {tb.shape[0]}x{tb.shape[1]}"
        )
    m, k = ta.shape
    n = tb.shape[1]
    out = torch.empty((m, n), dtype=torch.float64, device=dev)
    # Strided operands go straight to the kernel: a transposed view costs no copy.
    N.check(N.load().bb_matmul_f64(ta.data_ptr(), ta.stride(0), ta.stride(1), tb.data_ptr(), tb.stride(0),
                                   tb.stride(1), out.data_ptr(), m, n, k, _stream(dev)))
    return _ret(out, host)


def row_logsumexp(s):
    """numerics.py:48-59: per-row logsumexp with max subtraction; all -inf rows give -inf."""
    dev, host = _dev_of(s), _host_out(s)
    t = _as(s, 2, "row_logsumexp input", dev)
    if t.numel() == 0:
        raise ValueError("row_logsumexp requires a nonempty matrix")
    t = t if t.stride(1) == 1 else t.contiguous()
    out = torch.empty(t.shape[0], dtype=torch.float64, device=dev)
    N.check(N.load().bb_row_logsumexp_f64(t.data_ptr(), t.shape[0], t.shape[1], t.stride(0), out.data_ptr(),
                                          _stream(dev)))
    return _ret(out, host)


def lse_merge(a, b):
    """numerics.py:62-69: elementwise log(exp(a) + exp(b)) with np.logaddexp's semantics."""
    dev, host = _dev_of(a, b), _host_out(a, b)
    ta, tb = _as(a, 1, "lse_merge operand a", dev), _as(b, 1, "lse_merge operand b", dev)
    if ta.shape != tb.shape:
        raise ValueError(f"lse_merge length mismatch: {ta.shape[0]} vs {tb.shape[0]}")
    ta, tb = ta.contiguous(), tb.contiguous()
    out = torch.empty_like(ta)
    N.check(N.load().bb_lse_merge_f64(ta.data_ptr(), tb.data_ptr(), out.data_ptr(), ta.numel(), _stream(dev)))
    return _ret(out, host)


def exp_shifted(s, lse):
    """numerics.py:101-107: exp(s - lse[:, None]); rows with lse == -inf give exact zeros."""
    dev, host = _dev_of(s, lse), _host_out(s, lse)
    ts, tl = _as(s, 2, "exp_shifted input", dev).contiguous(), _as(lse, 1, "exp_shifted lse", dev).contiguous()
    if tl.shape[0] != ts.shape[0]:
        raise ValueError(f"exp_shifted: lse has {tl.shape[0]} entries for {ts.shape[0]} rows")
    out = torch.empty_like(ts)
    N.check(N.load().bb_exp_shifted_f64(ts.data_ptr(), tl.data_ptr(), out.data_ptr(), ts.shape[0], ts.shape[1],
                                        _stream(dev)))
    return _ret(out, host)


def exp_gap(a, b):
    """numerics.py:110-116: elementwise exp(a - b) with exp(-inf - anything) == 0."""
    dev, host = _dev_of(a, b), _host_out(a, b)
    ta = _as(a, 1, "exp_gap operand a", dev).contiguous()
    tb = _as(b, 1, "exp_gap operand b", dev).contiguous()
    if ta.shape != tb.shape:
        raise ValueError(f"exp_gap length mismatch: {ta.shape[0]} vs {tb.shape[0]}")
    out = torch.empty_like(ta)
    N.check(N.load().bb_exp_gap_f64(ta.data_ptr(), tb.data_ptr(), out.data_ptr(), ta.numel(), _stream(dev)))
    return _ret(out, host)


def row_softmax(s):
    """numerics.py:72-83: exp(s - row_logsumexp(s)); a fully masked row is an error."""
    dev, host = _dev_of(s), _host_out(s)
    t = _as(s, 2, "row_softmax input", dev).contiguous()
    lse = row_logsumexp(t)
    empty = torch.nonzero(lse == NEG_INF)
    if empty.numel():
        raise ValueError(f"row_softmax: row {int(empty[0, 0])} is fully masked (all -inf)")
    return _ret(exp_shifted(t, lse), host)


def rowsum_hadamard(a, b):
    """numerics.py:86-92: out[i] = sum_j a[i, j] * b[i, j]."""
    dev, host = _dev_of(a, b), _host_out(a, b)
    ta = _as(a, 2, "rowsum_hadamard operand a", dev).contiguous()
    tb = _as(b, 2, "rowsum_hadamard operand b", dev).contiguous()
    if ta.shape != tb.shape:
        raise ValueError(f"rowsum_hadamard shape mismatch: {tuple(ta.shape)} vs {tuple(tb.shape)}")
    out = torch.empty(ta.shape[0], dtype=torch.float64, device=dev)
    N.check(N.load().bb_rowsum_hadamard_f64(ta.data_ptr(), tb.data_ptr(), out.data_ptr(), ta.shape[0], ta.shape[1],
                                            _stream(dev)))
    return _ret(out, host)


def seeded_random_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """numerics.py:95-98: entries U[-1, 1] from PCG64(seed) -- the reference's test inputs."""
    return np.random.Generator(np.random.PCG64(seed)).uniform(-1.0, 1.0, size=(rows, cols))


def softmax_xent(logits, lse, targets):
    """loss[r] = lse[r] - logits[r, y_r] and g = softmax - onehot(y) (oracle.py:146-150), one pass."""
    dev = logits.device
    rows, vocab = logits.shape
    loss = torch.empty(rows, dtype=torch.float64, device=dev)
    g = torch.empty_like(logits)
    N.check(N.load().bb_xent_f64(logits.data_ptr(), lse.data_ptr(), targets.data_ptr(), rows, vocab,
                                 loss.data_ptr(), g.data_ptr(), _stream(dev)))
    return loss, g
