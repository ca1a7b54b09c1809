"""Host-side checks of layer.py (no GPU): AttentionParams validation mirrors oracle.py:38-44."""

import numpy as np
import pytest

from paper_2509_19836_b200.layer import AttentionParams


def test_non_square_params_rejected():
    with pytest.raises(ValueError, match="w_q must be 3x3"):
        AttentionParams(dim=3, w_q=np.zeros((3, 2)), w_k=np.zeros((3, 3)), w_v=np.zeros((3, 3)), w_attn=np.zeros((3, 3)))


def test_square_params_accepted():
    p = AttentionParams(dim=2, w_q=np.eye(2), w_k=np.eye(2), w_v=np.eye(2), w_attn=np.eye(2))
    assert p.dim == 2


@pytest.mark.parametrize("kind,n,g,bl", [("zigzag", 64, 4, None), ("striped", 48, 3, None), ("block_striped", 64, 2, 8),
                                         ("contiguous", 16, 2, None)])
def test_shard_row_map_inverts_the_shard_gather(kind, n, g, bl):
    """The row map the projection GEMM stores through sends token row r to the shard-major row
    that shard_rows' gather reads it from (bit-exact against the golden-pinned layouts)."""
    from paper_2509_19836_b200.layer import shard_row_map
    from paper_2509_19836_b200.partitioning import ShardLayout, shard_token_arrays

    layout = ShardLayout(kind, n, g, bl)
    rmap = shard_row_map(layout)
    shard_major = np.concatenate([np.asarray(ids) - 1 for ids in shard_token_arrays(layout)])
    assert sorted(rmap.tolist()) == list(range(n))
    assert np.array_equal(rmap[shard_major], np.arange(n))


def test_attention_backward_checks_shapes_before_the_device():
    """The reference raises for these through masked_scores / its matmuls (oracle.py:66-75,
    98-119); the kernel path must raise before reading device memory out of bounds."""
    from paper_2509_19836_b200.layer import attention_backward
    from paper_2509_19836_b200.masks import block_sparse_mask, causal_mask

    q, k, v, o, do = (np.zeros((8, 16)) for _ in range(5))
    lse = np.zeros(8)
    with pytest.raises(ValueError, match="Q has dim 16 but K has dim 8"):
        attention_backward(q, np.zeros((8, 8)), v, o, lse, do, causal_mask())
    with pytest.raises(ValueError, match="K has 8 rows but V has 4"):
        attention_backward(q, k, np.zeros((4, 16)), o, lse, do, causal_mask())
    with pytest.raises(ValueError, match="O must be 8x16"):
        attention_backward(q, k, v, np.zeros((4, 16)), lse, do, causal_mask())
    with pytest.raises(ValueError, match="lse must have 8 entries"):
        attention_backward(q, k, v, o, np.zeros(5), do, causal_mask())
    with pytest.raises(ValueError, match="block_mask must be 2x2"):  # mask smaller than the sequence
        attention_backward(q, k, v, o, lse, do, block_sparse_mask(np.ones((1, 1)), 4))


def test_hostio_out_arrays():
    """to_host_f64 fills a preallocated float64 result (backward_grads pages it in early) and
    rejects one of the wrong shape / dtype / layout."""
    import numpy as np
    import pytest
    import torch

    from paper_2509_19836_b200 import hostio

    t = torch.arange(24, dtype=torch.float32).reshape(2, 3, 4) / 7
    out = hostio.empty_f64(t)
    assert out.shape == (2, 3, 4) and out.dtype == np.float64 and not out.any()
    res = hostio.to_host_f64(t, out)
    assert res is out and np.array_equal(out, t.double().numpy())
    for bad in (np.empty((2, 3, 5)), np.empty((2, 3, 4), dtype=np.float32), np.empty((4, 3, 2)).transpose(2, 1, 0)):
        with pytest.raises(ValueError):
            hostio.to_host_f64(t, bad)
