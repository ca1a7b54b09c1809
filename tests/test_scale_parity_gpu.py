"""Parity on BASELINE.json's own configurations (not just the small grids of
test_parity_gpu.py):

* cfg1 exactly -- N = 4096, G = 4 simulated ranks, 8 heads, d = 64, causal; zigzag (burst and
  ring backward), contiguous and striped (burst) -- against the CPU oracle
  (oracle/burst_oracle.py, pinned to burstsim's golden vectors), with the tolerances of
  test_parity_gpu.py.
* cfg2 (128K tokens, causal, 32 heads, d = 128) and cfg4 (512K tokens, GQA 32q/8kv, sliding
  window 32K AND 128K causal documents at 2048-token blocks, block_striped) at full size on one
  GPU: 1024-4096 key tiles of lazy rescale and fp32 accumulation per row.  The fp64 numpy
  oracle cannot run these sizes, so sampled rows are checked against the same math in float64
  on the GPU (torch): O / lse for 256 query rows x 2 heads, dQ for those rows, dK / dV for 256
  key rows of their kv heads (summed over the GQA group's query heads, as the kernel does).  lse and D = rowsum(dO o O) enter the sampled dK / dV through every query, so they
  are recomputed in float64 for the whole sequence of the sampled heads.
"""

import math
import multiprocessing as mp
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest
import torch

import paper_2509_19836_b200 as bb
from oracle import burst_oracle as O
from paper_2509_19836_b200.partitioning import device_token_ids

pytestmark = pytest.mark.gpu

TOL_O, TOL_LSE, TOL_G = 1e-2, 2e-3, 1e-2


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-12))


def _oracle_case(args):
    q, k, v, do, layout, backward = args
    return O.mh_ring_attention(q, k, v, do, layout, ("causal", None, None, None), O.ring_visit(1, 4), backward=backward)


def test_cfg1_exact_config_matches_oracle(cuda):
    n, g, h, d = 4096, 4, 8, 64
    rng = np.random.default_rng(4096)

    def quant(shape):
        t = torch.from_numpy(rng.uniform(-1, 1, shape)).float().to(torch.bfloat16)
        return t, t.double().numpy()

    (qt, q), (kt, k), (vt, v), (dot, do) = (quant((n, h, d)) for _ in range(4))
    cases = [("zigzag", "burst"), ("zigzag", "ring"), ("contiguous", "burst"), ("striped", "burst")]
    with ProcessPoolExecutor(max_workers=4, mp_context=mp.get_context("fork")) as ex:  # numpy-only workers
        refs = list(ex.map(_oracle_case, [(q, k, v, do, (kind, n, g, None), bw) for kind, bw in cases]))
    for (kind, backward), ref in zip(cases, refs):
        layout = bb.ShardLayout(kind, n, g)
        st = bb.make_device_states(layout, qt, kt, vt, devices=["cuda:0"] * g)
        bb.distributed_forward(st, layout, bb.causal_mask())
        (bb.burst_backward if backward == "burst" else bb.ring_backward)(st, bb.shard_rows(layout, dot), layout,
                                                                           bb.causal_mask())
        o = bb.gather_rows(layout, [s.o for s in st]).double().cpu().numpy()
        lse = bb.gather_rows(layout, [s.lse.t().contiguous() for s in st]).double().cpu().numpy().T
        assert np.max(np.abs(o - ref["o"])) < TOL_O, kind
        assert np.max(np.abs(lse - ref["lse"])) < TOL_LSE, kind
        for name in ("dq", "dk", "dv"):
            got = bb.gather_rows(layout, [getattr(s, name) for s in st]).double().cpu().numpy()
            assert rel(got, ref[name]) < TOL_G, (kind, backward, name)


# ------------------------------------------------------------------ sampled rows at scale
def _fp64_reference(q, k, v, do, allowed, key_span, rows, cols, scale, chunk):
    """Float64 attention of one (query head, kv head) pair on the GPU.

    q, do: [N, d]; k, v: [N, d] (fp64).  allowed(qi, ki) -> bool [len(qi), len(ki)] for 0-based
    token index tensors; key_span(q0, q1) -> (k0, k1) bounds every allowed key of those
    queries.  Returns O / lse / dQ of ``rows``, dK / dV of ``cols``.
    """
    n = q.shape[0]
    ar = torch.arange(n, device=q.device)
    lse = torch.full((n,), float("-inf"), dtype=torch.float64, device=q.device)
    dvec = torch.zeros(n, dtype=torch.float64, device=q.device)
    o_rows = torch.zeros(len(rows), q.shape[1], dtype=torch.float64, device=q.device)
    pos = {int(r): i for i, r in enumerate(rows)}
    for q0 in range(0, n, chunk):
        q1 = min(q0 + chunk, n)
        k0, k1 = key_span(q0, q1)
        s = (q[q0:q1] @ k[k0:k1].T) * scale
        s.masked_fill_(~allowed(ar[q0:q1], ar[k0:k1]), float("-inf"))
        l = torch.logsumexp(s, dim=1)
        p = torch.exp(s - l[:, None])
        p.nan_to_num_(0.0)
        o = p @ v[k0:k1]
        lse[q0:q1] = l
        dvec[q0:q1] = (do[q0:q1] * o).sum(1)
        for r in range(q0, q1):
            if r in pos:
                o_rows[pos[r]] = o[r - q0]
        del s, p, o
    rows_t = torch.as_tensor(rows, device=q.device)
    cols_t = torch.as_tensor(cols, device=q.device)
    # dQ of the sampled rows
    dq_rows = torch.zeros(len(rows), q.shape[1], dtype=torch.float64, device=q.device)
    for i, r in enumerate(rows):
        k0, k1 = key_span(int(r), int(r) + 1)
        s = (q[r:r + 1] @ k[k0:k1].T) * scale
        s.masked_fill_(~allowed(ar[r:r + 1], ar[k0:k1]), float("-inf"))
        p = torch.exp(s - lse[r]).nan_to_num_(0.0)
        ds = p * (do[r:r + 1] @ v[k0:k1].T - dvec[r])
        dq_rows[i] = (ds @ k[k0:k1])[0] * scale
    # dK / dV of the sampled key rows: every query that can see them
    dk_cols = torch.zeros(len(cols), q.shape[1], dtype=torch.float64, device=q.device)
    dv_cols = torch.zeros_like(dk_cols)
    for q0 in range(0, n, chunk):
        q1 = min(q0 + chunk, n)
        s = (q[q0:q1] @ k[cols_t].T) * scale
        ok = allowed(ar[q0:q1], cols_t)
        if not ok.any():
            continue
        s.masked_fill_(~ok, float("-inf"))
        p = torch.exp(s - lse[q0:q1, None]).nan_to_num_(0.0)
        ds = p * (do[q0:q1] @ v[cols_t].T - dvec[q0:q1, None])
        dk_cols += (ds.T @ q[q0:q1]) * scale
        dv_cols += p.T @ do[q0:q1]
    return o_rows, lse[rows_t], dq_rows, dk_cols, dv_cols


def _run_scale_case(layout, mask, n, hq, hkv, d, allowed, key_span, heads, seed):
    dev = torch.device("cuda:0")
    gen = torch.Generator(device=dev).manual_seed(seed)

    def rnd(h):
        return (torch.rand(n, h, d, device=dev, generator=gen) * 2 - 1).to(torch.bfloat16)

    q, k, v, do = rnd(hq), rnd(hkv), rnd(hkv), rnd(hq)
    st = bb.make_device_states(layout, q, k, v, devices=["cuda:0"])
    bb.distributed_forward(st, layout, mask)
    bb.burst_backward(st, bb.shard_rows(layout, do), layout, mask)
    s0 = st[0]
    ids = device_token_ids(layout, 1) - 1  # shard row r holds token ids[r]
    inv = np.empty(n, dtype=np.int64)
    inv[ids] = np.arange(n)
    rng = np.random.default_rng(seed)
    rows = np.unique(np.concatenate([[0, n - 1], rng.choice(n, 254, replace=False)]))
    cols = np.unique(np.concatenate([[0, n - 1], rng.choice(n, 254, replace=False)]))
    scale = 1 / math.sqrt(d)
    group = hq // hkv
    r_sh, c_sh = torch.as_tensor(inv[rows], device=dev), torch.as_tensor(inv[cols], device=dev)
    for kvh in sorted({h // group for h in heads}):
        dk_ref = dv_ref = 0
        for h in range(kvh * group, (kvh + 1) * group):  # dK / dV sum over the GQA group's query heads
            ref = _fp64_reference(q[:, h].double(), k[:, kvh].double(), v[:, kvh].double(), do[:, h].double(),
                                  allowed, key_span, rows, cols, scale, chunk=2048)
            dk_ref, dv_ref = dk_ref + ref[3], dv_ref + ref[4]
            if h not in heads:
                continue
            o = s0.o[r_sh, h, :d].double()
            lse = s0.lse[h, r_sh].double()
            assert float((o - ref[0]).abs().max()) < TOL_O, h
            assert float((lse - ref[1]).abs().max()) < TOL_LSE, h
            err = float(torch.linalg.norm(s0.dq[r_sh, h, :d].double() - ref[2]) / torch.linalg.norm(ref[2]))
            assert err < TOL_G, (h, "dq", err)
        for got, want, name in ((s0.dk[c_sh, kvh, :d], dk_ref, "dk"), (s0.dv[c_sh, kvh, :d], dv_ref, "dv")):
            err = float(torch.linalg.norm(got.double() - want) / torch.linalg.norm(want))
            assert err < TOL_G, (kvh, name, err)
    del st, q, k, v, do
    torch.cuda.empty_cache()


def test_cfg2_128k_causal_sampled_rows(cuda):
    n = 131072
    layout = bb.ShardLayout("zigzag", n, 1)

    def allowed(qi, ki):
        return ki[None, :] <= qi[:, None]

    _run_scale_case(layout, bb.causal_mask(), n, 32, 32, 128, allowed, lambda q0, q1: (0, q1), heads=(0, 21), seed=2)


def test_cfg4_512k_gqa_swa_doc_sampled_rows(cuda):
    n, bl, window, doc = 524288, 2048, 32768, 131072
    band = bb.block_mask_from_window(n, bl, window).block_mask
    docs = bb.document_mask([doc] * (n // doc), bl).block_mask
    mask = bb.block_sparse_mask(np.logical_and(band, docs).astype(np.int64), bl)
    bm = torch.from_numpy(np.asarray(mask.block_mask) != 0).cuda()
    layout = bb.ShardLayout("block_striped", n, 1, bl)

    def allowed(qi, ki):
        return bm[(qi // bl)[:, None], (ki // bl)[None, :]]

    def key_span(q0, q1):  # the band is block-granular: a query sees its whole own block
        return max(0, (q0 // bl - window // bl + 1) * bl), min(n, -(-q1 // bl) * bl)

    _run_scale_case(layout, mask, n, 32, 8, 128, allowed, key_span, heads=(0, 29), seed=4)
