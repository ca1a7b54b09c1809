"""Kernel-level numerics on the B200: each C-ABI kernel against a plain PyTorch
fp32 computation on the same bf16-quantised inputs.  (End-to-end parity with the
fp64 oracle lives in test_parity_gpu.py.)"""

import math

import numpy as np
import pytest
import torch

from paper_2509_19836_b200 import kernels as K
from paper_2509_19836_b200.masks import block_sparse_mask, causal_mask, full_mask, sliding_window_mask
from paper_2509_19836_b200.partitioning import ShardLayout, device_token_ids

pytestmark = pytest.mark.gpu


def _ref_attention(q, k, v, allowed, scale):
    """fp32 reference for one (query shard, key shard) pair, GQA by head repetition."""
    hq, hkv = q.shape[1], k.shape[1]
    rep = hq // hkv
    qf, kf, vf = q.float(), k.float().repeat_interleave(rep, 1), v.float().repeat_interleave(rep, 1)
    s = torch.einsum("qhd,khd->hqk", qf, kf) * scale
    s = s.masked_fill(~allowed[None], float("-inf"))
    lse = torch.logsumexp(s, dim=-1)  # [h, q]
    p = torch.exp(s - lse[..., None]).nan_to_num(0.0)
    o = torch.einsum("hqk,khd->qhd", p, vf)
    return o, lse


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("m,n,k", [(128, 256, 64), (304, 520, 200), (640, 1000, 320), (1024, 768, 4096)])
def test_gemm_matches_torch(cuda, a_mn, b_mn, m, n, k):
    g = torch.Generator(device=cuda).manual_seed(m + n + k)
    a = torch.randn(m, k, device=cuda, generator=g).to(torch.bfloat16)
    b = torch.randn(n, k, device=cuda, generator=g).to(torch.bfloat16)
    a_st = a.t().contiguous() if a_mn else a
    b_st = b.t().contiguous() if b_mn else b
    c = torch.zeros(m, n, device=cuda)
    K.gemm(a_st, b_st, c, m, n, k, a_mn, b_mn, accumulate=False)
    ref = a.float() @ b.float().t()
    torch.cuda.synchronize()
    err = (c - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-3, err
    K.gemm(a_st, b_st, c, m, n, k, a_mn, b_mn, accumulate=True)
    err2 = (c - 2 * ref).abs().max().item() / ref.abs().max().item()
    assert err2 < 1e-3, err2


MASKS = {
    "full": lambda n: full_mask(),
    "causal": lambda n: causal_mask(),
    "window": lambda n: sliding_window_mask(max(1, n // 3)),
    "block": lambda n: block_sparse_mask(np.tril(np.ones((4, 4), dtype=np.int64)) - np.eye(4, k=-2, dtype=np.int64), n // 4),
}


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("maskname", list(MASKS))
@pytest.mark.parametrize("n,hq,hkv", [(512, 2, 2), (300, 4, 2)])
def test_fwd_single_step_matches_torch(cuda, d, maskname, n, hq, hkv):
    torch.manual_seed(0)
    mask = MASKS[maskname](n)
    layout = ShardLayout("contiguous", n, 1)
    q = torch.randn(n, hq, d, device=cuda).to(torch.bfloat16)
    k = torch.randn(n, hkv, d, device=cuda).to(torch.bfloat16)
    v = torch.randn(n, hkv, d, device=cuda).to(torch.bfloat16)
    o = torch.zeros(n, hq, d, device=cuda)
    lse = torch.full((hq, n), float("-inf"), device=cuda)
    scale = 1.0 / math.sqrt(d)
    dm = K.device_mask(mask, cuda)
    K.attn_fwd_step(q, k, v, o, lse, layout, dm, 1, 1, scale)
    ids = torch.from_numpy(device_token_ids(layout, 1)).to(cuda)
    from paper_2509_19836_b200.masks import allowed_pairs

    allowed = torch.from_numpy(allowed_pairs(mask, ids.cpu().numpy(), ids.cpu().numpy())).to(cuda)
    o_ref, lse_ref = _ref_attention(q, k, v, allowed, scale)
    torch.cuda.synchronize()
    live = torch.isfinite(lse_ref)
    assert torch.equal(torch.isfinite(lse), live)
    assert (lse[live] - lse_ref[live]).abs().max().item() < 2e-3
    assert (o - o_ref).abs().max().item() < 1e-2


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("maskname", ["full", "causal", "window"])
def test_fwd_two_step_merge(cuda, d, maskname):
    """Two ring steps (zigzag, G=2) merged in the epilogue equal one softmax over both shards."""
    n, hq = 1024, 2
    mask = MASKS[maskname](n)
    layout = ShardLayout("zigzag", n, 2)
    torch.manual_seed(1)
    qg = torch.randn(n, hq, d, device=cuda).to(torch.bfloat16)
    kg = torch.randn(n, hq, d, device=cuda).to(torch.bfloat16)
    vg = torch.randn(n, hq, d, device=cuda).to(torch.bfloat16)
    idx = [torch.from_numpy(device_token_ids(layout, i) - 1).to(cuda) for i in (1, 2)]
    dm = K.device_mask(mask, cuda)
    scale = 1.0 / math.sqrt(d)
    from paper_2509_19836_b200.masks import allowed_pairs

    for i in (1, 2):
        qi = qg[idx[i - 1]].contiguous()
        o = torch.zeros(n // 2, hq, d, device=cuda)
        lse = torch.full((hq, n // 2), float("-inf"), device=cuda)
        for j in ((2, 1) if i == 1 else (1, 2)):  # flat ring visit order: own shard last
            K.attn_fwd_step(qi, kg[idx[j - 1]].contiguous(), vg[idx[j - 1]].contiguous(), o, lse, layout, dm, i, j, scale)
        allowed = torch.from_numpy(
            allowed_pairs(mask, device_token_ids(layout, i), np.arange(1, n + 1))
        ).to(cuda)
        o_ref, lse_ref = _ref_attention(qi, kg, vg, allowed, scale)
        torch.cuda.synchronize()
        assert (lse - lse_ref).abs().max().item() < 2e-3
        assert (o - o_ref).abs().max().item() < 1e-2


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("maskname", list(MASKS))
@pytest.mark.parametrize("n,hq,hkv", [(512, 2, 2), (300, 4, 2)])
def test_bwd_single_step_matches_autograd(cuda, d, maskname, n, hq, hkv):
    torch.manual_seed(2)
    mask = MASKS[maskname](n)
    layout = ShardLayout("contiguous", n, 1)
    q = torch.randn(n, hq, d, device=cuda).to(torch.bfloat16)
    k = torch.randn(n, hkv, d, device=cuda).to(torch.bfloat16)
    v = torch.randn(n, hkv, d, device=cuda).to(torch.bfloat16)
    do = torch.randn(n, hq, d, device=cuda).to(torch.bfloat16)
    scale = 1.0 / math.sqrt(d)
    dm = K.device_mask(mask, cuda)
    o = torch.zeros(n, hq, d, device=cuda)
    lse = torch.full((hq, n), float("-inf"), device=cuda)
    K.attn_fwd_step(q, k, v, o, lse, layout, dm, 1, 1, scale)
    delta = torch.empty(hq, n, device=cuda)
    K.bwd_preprocess(do, o, delta)
    dq = torch.zeros(n, hq, d, device=cuda)
    dk = torch.zeros(n, hkv, d, device=cuda)
    dv = torch.zeros(n, hkv, d, device=cuda)
    K.attn_bwd_step(q, k, v, do, lse, delta, dq, dk, dv, layout, dm, 1, 1, scale)
    from paper_2509_19836_b200.masks import allowed_pairs

    ids = device_token_ids(layout, 1)
    allowed = torch.from_numpy(allowed_pairs(mask, ids, ids)).to(cuda)
    live = allowed.any(1)  # rows with at least one key
    qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
    o_ref, _ = _ref_attention(qf, kf, vf, allowed, scale)
    (o_ref[live] * do.float()[live]).sum().backward()
    torch.cuda.synchronize()
    d_ref = (do.float() * o_ref).sum(-1).t()
    assert (delta[:, live] - d_ref[:, live]).abs().max().item() < 1e-2 * max(1.0, d_ref.abs().max().item())
    for got, want, name in ((dq, qf.grad, "dq"), (dk, kf.grad, "dk"), (dv, vf.grad, "dv")):
        rel = (got - want).norm().item() / max(want.norm().item(), 1e-6)
        assert rel < 1e-2, (name, rel)


@pytest.mark.parametrize("n,vocab,dim,rows_tile", [(300, 1000, 64, 128), (512, 4096, 256, 512), (256, 777, 128, 100)])
def test_lmhead_matches_torch(cuda, n, vocab, dim, rows_tile):
    torch.manual_seed(3)
    h = torch.rand(n, dim, device=cuda).mul(2).sub(1).to(torch.bfloat16)
    w = (torch.rand(vocab, dim, device=cuda).mul(2).sub(1) / math.sqrt(dim)).to(torch.bfloat16)
    y = torch.randint(0, vocab, (n,), device=cuda)
    loss = torch.empty(n, device=cuda)
    dh = torch.empty(n, dim, device=cuda)
    dw = torch.zeros(vocab, dim, device=cuda)
    ws = torch.empty(K.lmhead_workspace_bytes(n, vocab, dim, rows_tile), dtype=torch.uint8, device=cuda)
    K.lmhead_fused(h, w, y, loss, dh, dw, rows_tile, 64, ws)
    hf, wf = h.float().requires_grad_(), w.float().requires_grad_()
    logits = hf @ wf.t()
    ref = torch.nn.functional.cross_entropy(logits, y, reduction="none")
    ref.sum().backward()
    torch.cuda.synchronize()
    assert (loss - ref).abs().max().item() < 2e-3
    for got, want in ((dh, hf.grad), (dw, wf.grad)):
        assert (got - want).norm().item() / want.norm().item() < 1e-2


def test_bwd_kv_head_halves_equal_full_step():
    """bb_attn_bwd_step over kv-head ranges (the ring's split own step) sums to the full step for
    every (i, j) of a 4-way zigzag causal ring with GQA; run in a subprocess under a timeout so a
    kernel hang (seen with the 2-CTA multicast variant) fails instead of stalling the suite."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    res = subprocess.run([sys.executable, str(root / "tools" / "bwd_heads_check.py")], capture_output=True, text=True,
                         timeout=300, env=dict(os.environ, PYTHONPATH=str(root)))
    assert res.returncode == 0 and "OK" in res.stdout, res.stdout[-2000:] + res.stderr[-2000:]


def test_fill_and_fold_kernels(cuda):
    """bb_fill_u32 / bb_add_rows_f32 (the ring's accumulator initialisation and gradient
    folds): exact against torch, on whole tensors and on head-range views."""
    x = torch.empty(1000, 6, 36, device="cuda")
    assert bool(torch.isneginf(K.fill_(x, float("-inf"))).all())
    assert not K.fill_(x).any()
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(333, 8, 64, device="cuda", generator=g)
    b = torch.randn(333, 8, 64, device="cuda", generator=g)
    ref = a.clone()
    ref[:, 2:5] += b[:, 2:5]
    K.add_rows_(a[:, 2:5], b[:, 2:5])
    assert torch.equal(a, ref)
    ref += b
    K.add_rows_(a, b)
    assert torch.equal(a, ref)
    with pytest.raises(ValueError):
        K.add_rows_(a[:, :, :10], b[:, :, :10])  # rows are not contiguous runs
    y = torch.empty(7, 3, device="cuda")
    assert bool((K.fill_(y[1:], 2.5) == 2.5).all())  # odd count, 4-byte aligned start: word stores


def test_hostio_staged_copies_are_exact(cuda):
    """The drop-in API's host <-> device paths (pinned staging, chunked, threaded host casts):
    identical to the plain torch conversions, across chunk boundaries (> 128 MB) and ragged ends."""
    from paper_2509_19836_b200 import hostio

    rng = np.random.default_rng(3)
    for shape in ((3, 5, 7), (45_000_001,)):
        x = rng.standard_normal(shape)  # float64
        d = hostio.to_device(x, torch.device("cuda"))
        assert d.dtype == torch.float32 and torch.equal(d.cpu(), torch.from_numpy(x).float())
        b = hostio.to_device(x, torch.device("cuda"), torch.bfloat16)
        assert torch.equal(b.cpu(), torch.from_numpy(x).float().to(torch.bfloat16))
        h = hostio.to_host_f64(d)
        assert h.dtype == np.float64 and np.array_equal(h, x.astype(np.float32).astype(np.float64))
    assert hostio.to_host_f64(torch.empty(0, 4, device="cuda")).shape == (0, 4)


@pytest.mark.parametrize("kind,g", [("zigzag", 2), ("contiguous", 2), ("zigzag", 1)])
@pytest.mark.parametrize("maskname", ["causal", "window", "block"])
def test_oversized_shards_split_into_sub_shard_pairs(cuda, kind, g, maskname):
    """A shard larger than one launch takes (the kernels' 4096-tile class tables, 524288 rows)
    is run as the pairs of its consecutive-id sub-shards (bb_api.cu).  Forced here at 256 rows
    (bb_debug_set_split_rows): every ring step, a prefix (n_q < shard) and the bf16 O copy must
    match the single-launch results up to bf16 rounding of P and accumulation order."""
    n, h, d = 4096, 2, 64
    layout = ShardLayout(kind, n, g)
    mask = {"causal": causal_mask(), "window": sliding_window_mask(1000),
            "block": block_sparse_mask(np.tril(np.ones((16, 16), dtype=np.int64)) - np.tril(np.ones((16, 16), dtype=np.int64), -5), 256)}[maskname]
    dev = torch.device("cuda")
    dm = K.device_mask(mask, dev)
    m = layout.shard_size
    gen = torch.Generator(device=dev).manual_seed(9)
    q, k, v, do = ((torch.rand(g, m, h, d, device=dev, generator=gen) * 2 - 1).to(torch.bfloat16) for _ in range(4))
    scale = 1 / math.sqrt(d)

    def run(n_q):
        outs = []
        for i in range(g):
            o = torch.zeros(n_q, h, d, device=dev)
            lse = torch.full((h, n_q), float("-inf"), device=dev)
            o16 = torch.empty(n_q, h, d, dtype=torch.bfloat16, device=dev)
            for j in range(g):
                K.attn_fwd_step(q[i, :n_q].contiguous(), k[j], v[j], o, lse, layout, dm, i + 1, j + 1, scale, n_q=n_q,
                                o_bf16=o16 if j == g - 1 else None)
            assert torch.equal(o16, o.to(torch.bfloat16))
            delta = torch.empty(h, n_q, device=dev)
            dq = torch.zeros(n_q, h, d, device=dev)
            dk, dv = torch.zeros(m, h, d, device=dev), torch.zeros(m, h, d, device=dev)
            K.bwd_preprocess(do[i, :n_q].contiguous(), o, delta)
            for j in range(g):
                dkj, dvj = torch.zeros(m, h, d, device=dev), torch.zeros(m, h, d, device=dev)
                K.attn_bwd_step(q[i, :n_q].contiguous(), k[j], v[j], do[i, :n_q].contiguous(), lse, delta, dq, dkj, dvj,
                                layout, dm, i + 1, j + 1, scale)
                dk += dkj
                dv += dvj
            outs.append((o, lse, dq, dk, dv))
        return outs

    for n_q in (m, 1000):
        ref = run(n_q)
        try:
            K.set_split_rows(256)
            got = run(n_q)
        finally:
            K.set_split_rows(0)
        for a, b in zip(got, ref):
            for x, y, name in zip(a, b, ("o", "lse", "dq", "dk", "dv")):
                fin = torch.isfinite(y)
                assert torch.equal(torch.isfinite(x), fin), name
                err = float((x[fin] - y[fin]).abs().max()) / max(float(y[fin].abs().max()), 1e-30)
                # P is rounded to bf16 against each launch's own running max, so O and the
                # gradients move at bf16 level (as between a ring step and one big step); the
                # fp32 statistics (lse) only by summation order
                assert err < (1e-5 if name == "lse" else 8e-3), (name, n_q, err)  # 8e-3: two bf16 ulps
