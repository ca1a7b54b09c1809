"""burstsim.oracle's layer entry points on the GPU (paper_2509_19836_b200.layer) against the CPU
oracle: project_qkv, the permutation-fused project_qkv_shards (bit-exact against projecting
then gathering), attention_forward / attention_backward (bf16 tolerances)."""

import numpy as np
import pytest
import torch

from oracle import burst_oracle as O
from paper_2509_19836_b200 import layer as Lyr
from paper_2509_19836_b200.masks import block_sparse_mask, causal_mask, full_mask, sliding_window_mask
from paper_2509_19836_b200.partitioning import ShardLayout, device_token_ids

pytestmark = pytest.mark.gpu


def _bf16(a):
    return torch.from_numpy(a).float().to(torch.bfloat16).double().numpy()


def _params(d, seed=0):
    rng = np.random.default_rng(seed)
    w = [_bf16(rng.uniform(-1, 1, (d, d)) / np.sqrt(d)) for _ in range(4)]
    return Lyr.AttentionParams(d, *w)


@pytest.mark.parametrize("n,d", [(256, 64), (1000, 128), (77, 40)])
def test_project_qkv_matches_matmul(n, d):
    p = _params(d)
    x = _bf16(np.random.default_rng(1).uniform(-1, 1, (n, d)))
    q, k, v = Lyr.project_qkv(x, p)
    for got, w in zip((q, k, v), (p.w_q, p.w_k, p.w_v)):
        want = x @ w
        assert got.shape == want.shape
        assert np.abs(got - want).max() <= 1e-2 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("kind,g,block", [("zigzag", 4, None), ("striped", 2, None), ("block_striped", 4, 64)])
def test_project_qkv_shards_is_the_permuted_projection(kind, g, block):
    n, d, heads = 2048, 128, 2
    p = _params(d, 3)
    x = _bf16(np.random.default_rng(2).uniform(-1, 1, (n, d)))
    layout = ShardLayout(kind, n, g, block)
    shards = Lyr.project_qkv_shards(x, p, layout, heads=heads)
    full = Lyr.project_qkv(torch.from_numpy(x).cuda(), p)  # identity row map, same GEMM tiles
    for i, (qi, ki, vi) in enumerate(shards):
        rows = torch.from_numpy(device_token_ids(layout, i + 1) - 1).cuda()
        for got, f in zip((qi, ki, vi), full):
            assert got.shape == (n // g, heads, d // heads) and got.is_contiguous()
            assert torch.equal(got.reshape(n // g, d), f.index_select(0, rows))  # bit-exact


@pytest.mark.parametrize("mname", ["causal", "full", "window", "block"])
@pytest.mark.parametrize("nq,nk,d", [(512, 512, 128), (300, 300, 64), (200, 384, 96), (384, 200, 64)])
def test_attention_forward_backward_match_oracle(mname, nq, nk, d):
    """Any nq, nk (oracle.py:80-119 takes both): the kernels run on one shard of max(nq, nk)
    ids with queries and keys as its leading rows."""
    if mname == "window" and nq > nk:
        pytest.skip("rows past nk + w have no key: covered by test_attention_forward_errors")
    rng = np.random.default_rng(5)
    q, do = (_bf16(rng.uniform(-1, 1, (nq, d))) for _ in range(2))
    k, v = (_bf16(rng.uniform(-1, 1, (nk, d))) for _ in range(2))
    n = max(nq, nk)
    if mname == "block":
        bl = 64 if n % 64 == 0 else 60
        nb = -(-n // bl)
        bm = np.tril(np.ones((nb, nb), dtype=np.int64))
        mask = block_sparse_mask(bm, bl)
        dense = np.kron(bm, np.ones((bl, bl)))[:nq, :nk] != 0
    else:
        mask = {"causal": causal_mask(), "full": full_mask(), "window": sliding_window_mask(50)}[mname]
        mt = {"causal": ("causal", None, None, None), "full": ("full", None, None, None),
              "window": ("sliding_window", 50, None, None)}[mname]
        dense = O.allowed(mt, np.arange(1, nq + 1), np.arange(1, nk + 1))
    o_ref, lse_ref = O.attention_forward(q, k, v, dense)
    res = Lyr.attention_forward(q, k, v, mask)
    assert np.abs(res.o - o_ref).max() < 1e-2
    assert np.abs(res.lse - lse_ref).max() < 2e-3
    dq_ref, dk_ref, dv_ref = O.attention_backward(q, k, v, o_ref, lse_ref, do, dense)
    gr = Lyr.attention_backward(q, k, v, res.o, res.lse, do, mask)
    for got, want in ((gr.dq, dq_ref), (gr.dk, dk_ref), (gr.dv, dv_ref)):
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-2


def test_attention_forward_errors():
    q = np.zeros((8, 16))
    with pytest.raises(ValueError, match="K has 8 rows but V has 4"):
        Lyr.attention_forward(q, q, np.zeros((4, 16)), causal_mask())
    bm = np.array([[0, 0], [1, 1]])
    with pytest.raises(ValueError, match="query row 1 has no unmasked key"):
        Lyr.attention_forward(q, q, q, block_sparse_mask(bm, 4))
    with pytest.raises(ValueError, match="query row 13 has no unmasked key"):  # 13 - 8 >= w = 5
        Lyr.attention_forward(np.zeros((16, 16)), q, q, sliding_window_mask(5))


def test_project_qkv_reference_cases():
    """The reference's TestProjectQkv (tests/test_oracle.py:56-95) at bf16 precision: identity
    weights return the (bf16-rounded) input, zero input gives zeros."""
    from oracle.burst_oracle import seeded_random_matrix

    d = 3
    eye = np.eye(d)
    x = seeded_random_matrix(5, d, 1)
    q, k, v = Lyr.project_qkv(x, Lyr.AttentionParams(dim=d, w_q=eye, w_k=eye, w_v=eye, w_attn=eye))
    for t in (q, k, v):
        assert np.array_equal(t, _bf16(x))
    p = Lyr.AttentionParams(2, *(seeded_random_matrix(2, 2, s) for s in (2, 3, 4)), np.eye(2))
    q, k, v = Lyr.project_qkv(np.zeros((4, 2)), p)
    assert not q.any() and not k.any() and not v.any()


@pytest.mark.parametrize("kind", ["zigzag", "striped"])
def test_projected_shards_feed_the_ring_kernels(kind):
    """X -> project_qkv_shards (permutation fused into the GEMM store) -> ring forward steps on
    the shards (all (i, j) pairs of a G=4 ring, one GPU) == attention of the projected sequence."""
    import math

    from paper_2509_19836_b200 import kernels as K

    n, d, g = 2048, 128, 4
    p = _params(d, 7)
    x = _bf16(np.random.default_rng(8).uniform(-1, 1, (n, d)))
    layout = ShardLayout(kind, n, g)
    shards = Lyr.project_qkv_shards(x, p, layout)
    dm = K.device_mask(causal_mask(), torch.device("cuda"))
    ref_q, ref_k, ref_v = (_bf16(x @ w) for w in (p.w_q, p.w_k, p.w_v))
    o_ref, lse_ref = O.attention_forward(ref_q, ref_k, ref_v, O.allowed(("causal", None, None, None),
                                                                         np.arange(1, n + 1), np.arange(1, n + 1)))
    for i in range(g):
        qi = shards[i][0]
        o = torch.zeros(n // g, 1, d, device="cuda")
        lse = torch.full((1, n // g), float("-inf"), device="cuda")
        for j in range(g):
            K.attn_fwd_step(qi, shards[j][1], shards[j][2], o, lse, layout, dm, i + 1, j + 1, 1.0 / math.sqrt(d))
        rows = device_token_ids(layout, i + 1) - 1
        assert np.abs(o[:, 0].double().cpu().numpy() - o_ref[rows]).max() < 1e-2
        assert np.abs(lse[0].double().cpu().numpy() - lse_ref[rows]).max() < 2e-3


@pytest.mark.parametrize("kind,heads,d", [("zigzag", 2, 64), ("block_striped", 2, 100), ("striped", 4, 128)])
def test_output_projection_of_the_ring_forward(kind, heads, d):
    """O W_attn (AttentionParams.w_attn): the forward's last step stores bf16(O)
    (bit-exact against casting the fp32 O it just merged), and project_output_shards writes
    bf16(O) W_attn back in global token order from the shards -- against the same product in
    float64 on the host, and identical whether it starts from the fused bf16 copy or casts O."""
    import paper_2509_19836_b200 as bb

    n, g = 2048, 4
    dim = heads * d
    layout = ShardLayout(kind, n, g, 64 if kind == "block_striped" else None)
    rng = np.random.default_rng(dim)
    q, k, v = (rng.uniform(-1, 1, (n, heads, d)) for _ in range(3))
    p = _params(dim, 11)
    st = bb.make_device_states(layout, q, k, v, devices=["cuda:0"] * g)
    bb.distributed_forward(st, layout, causal_mask(), emit_o_bf16=True)
    for s in st:
        assert torch.equal(s.o16, s.o.to(torch.bfloat16))
    out = bb.project_output_shards(st, p, layout)
    assert out.shape == (n, dim) and out.dtype == torch.bfloat16
    o_glob = bb.gather_rows(layout, [s.o16 for s in st]).double().cpu().numpy()[..., :d].reshape(n, dim)
    ref = o_glob @ np.asarray(p.w_attn)
    got = out.double().cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-2 * np.abs(ref).max()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 4e-3
    out32 = bb.project_output_shards([s.o for s in st], p, layout)
    assert torch.equal(out32, out)
