"""CPU-side checks of the C ABI: the sm_100a library loads on a GPU-less host,
exports exactly what include/burst_b200.h declares, validates arguments before
touching CUDA, and the product path refuses to run without the GPU (no CPU
fallback)."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2509_19836_b200 import _native as N
from paper_2509_19836_b200 import kernels as K

HEADER = Path(__file__).resolve().parent.parent / "include" / "burst_b200.h"


def declared_functions():
    text = HEADER.read_text()
    return set(re.findall(r"^\s*(?:int|int32_t|int64_t|const char\*)\s+(bb_\w+)\s*\(", text, re.M))


def test_library_exports_every_declared_symbol():
    lib = N.load()
    names = declared_functions()
    assert names == set(N.EXPORTS)
    for name in names:
        assert hasattr(lib, name), name
    assert lib.bb_abi_version() == 1


def test_library_is_sm100a_only():
    so = N.LIB_PATH.read_bytes()
    assert b"sm_100a" in so or b"sm_100" in so


def _bad_fwd_args(**over):
    a = N.BbAttnFwdArgs(n_q=8, n_k=8, hq=2, hkv=2, head_dim=64, softmax_scale=0.125, q_device=1, k_device=1)
    a.layout = N.BbLayout(kind=0, devices=1, seq_len=8, block_len=0)
    a.mask = N.BbMask(kind=1)
    for k, v in over.items():
        setattr(a, k, v)
    return a


@pytest.mark.parametrize(
    "over,msg",
    [
        ({"hq": 3}, "multiple of hkv"),
        ({"head_dim": 96}, "head_dim"),
        ({"q_device": 2}, "device indices"),
        ({"n_k": 16}, "shard sizes"),
        ({"n_q": 9}, "shard sizes"),
        ({"layout": N.BbLayout(kind=1, devices=3, seq_len=9, block_len=0)}, "zigzag"),
        ({"layout": N.BbLayout(kind=0, devices=3, seq_len=8, block_len=0)}, "divisible by 3 devices"),
        ({"layout": N.BbLayout(kind=3, devices=2, seq_len=8, block_len=0)}, "block_striped"),
        ({"layout": N.BbLayout(kind=3, devices=4, seq_len=8, block_len=2)}, "block_striped"),
        ({"mask": N.BbMask(kind=3, block_len=2, num_blocks=3, block_mask=8)}, "does not cover seq_len"),
        ({"mask": N.BbMask(kind=2, window=0)}, "sliding_window"),
    ],
)
def test_abi_validates_before_cuda(over, msg):
    lib = N.load()
    rc = lib.bb_attn_fwd_step(C.byref(_bad_fwd_args(**over)), None)
    assert rc != 0
    assert msg in lib.bb_last_error().decode()
    with pytest.raises((ValueError, RuntimeError), match=msg):
        N.check(rc)


def test_lmhead_abi_validation():
    lib = N.load()
    a = N.BbLmheadArgs(n=4, vocab=8, dim=8, rows_per_tile=0, vocab_per_tile=4)
    with pytest.raises(ValueError, match="tile sizes"):
        N.check(lib.bb_lmhead_fused(C.byref(a), None))


def test_no_cpu_fallback():
    from paper_2509_19836_b200.masks import causal_mask
    from paper_2509_19836_b200.partitioning import ShardLayout

    q = torch.zeros(8, 1, 64, dtype=torch.bfloat16)
    o = torch.zeros(8, 1, 64)
    lse = torch.zeros(1, 8)
    dm = K.DeviceMask(causal_mask(), N.BbMask(kind=1), None)
    with pytest.raises(ValueError, match="CUDA"):
        K.attn_fwd_step(q, q, q, o, lse, ShardLayout("contiguous", 8, 1), dm, 1, 1, 0.125)


def test_engine_refuses_without_gpu():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2509_19836_b200 import distributed as D
    from paper_2509_19836_b200.partitioning import ShardLayout

    x = np.zeros((8, 4))
    with pytest.raises(RuntimeError, match="CUDA"):
        D.make_device_states(ShardLayout("contiguous", 8, 2), x, x, x)


def test_product_never_imports_oracle():
    pkg = Path(N.__file__).resolve().parent
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\S+)", src, re.M), f
        assert "burst_oracle" not in src, f
