"""Sequence-sharded fused LM head + cross entropy (reference lmhead.py:41-93
is row-separable, so a 2^20-token job splits into per-GPU token shards with W replicated):
each rank runs the fused head on its own tokens, dW is summed over the shards (all_reduce_dw)
and the per-token losses are summed into the job's loss.

* gloo, world size 2, on CPU: the orchestration (shard split, dW all-reduce, loss all-reduce)
  with the per-shard head swapped for the oracle's fused_lmhead (a CPU test double, as in
  test_ring_gloo.py) must reproduce the unsharded oracle.
* NCCL on 2 GPUs (gpurun --gpus 2; skipped on one GPU): the same through the sm_100a kernels,
  against the fp64 oracle with the bf16 tolerances of test_parity_gpu.py.
"""

import math
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import burst_oracle as O

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(n=96, v=50, d=16, seed=3):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, (n, d)), rng.uniform(-1, 1, (v, d)) / math.sqrt(d), rng.integers(0, v, n)


def _oracle_shard(h, w_head, targets, cfg, device=None, dw_out=None):
    """CPU double of lmhead.fused_lmhead_loss for one shard (the oracle's fused head)."""
    from paper_2509_19836_b200.lmhead import FusedLossResult

    loss, dh, dw, peak = O.fused_lmhead(h.numpy(), w_head.numpy(), targets.numpy(), cfg.rows_per_tile, cfg.vocab_per_tile)
    dw_out[:, : dw.shape[1]] += torch.from_numpy(dw).to(dw_out.dtype)
    return FusedLossResult(loss=torch.from_numpy(loss), dh=torch.from_numpy(dh), dw=dw_out, peak_aux_elements=peak)


def _gloo_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_19836_b200 import lmhead as L

        L.fused_lmhead_loss = _oracle_shard
        h, w, y = _inputs()
        rows = np.array_split(np.arange(h.shape[0]), world)[rank]
        res = L.sharded_fused_lmhead_loss(torch.from_numpy(h[rows]), torch.from_numpy(w), torch.from_numpy(y[rows]),
                                          L.FusionConfig(16, 32))
        out_q.put((rank, rows, res.loss.numpy(), res.dh.numpy(), res.dw.double().numpy(), res.total_loss))
    finally:
        dist.destroy_process_group()


def test_sharded_head_orchestration_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [out_q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    h, w, y = _inputs()
    loss, dh, dw = O.naive_lmhead(h, w, y)
    for rank, rows, l_r, dh_r, dw_r, total in res:
        assert np.allclose(l_r, loss[rows], atol=1e-10)
        assert np.allclose(dh_r, dh[rows], atol=1e-10)
        assert np.allclose(dw_r, dw, atol=1e-5)  # dW all-reduced (fp32 accumulator) on every rank
        assert abs(total - loss.sum()) < 1e-8 * abs(loss.sum())


@pytest.mark.gpu
def test_sharded_head_two_gpus():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29711", str(ROOT / "tools" / "lmhead_shard_check.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "lmhead shard check ok" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("n,rows_tile", [(1000, 256), (512, 512)])
def test_fused_head_large_vocab_matches_fp64(cuda, n, rows_tile):
    """V = 128256 (LLaMA-3's ragged vocabulary: not a multiple of the 256-column UMMA tile),
    D = 4096, several row tiles (dW accumulates across them in fp32), against the same math in
    float64 on the GPU (the numpy oracle at this size would need 8 GB of fp64 logits)."""
    import paper_2509_19836_b200 as bb

    v, d = 128256, 4096
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(7)
    h = (torch.rand(n, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(v, d, device=dev, generator=g) * 2 - 1) / math.sqrt(d)).to(torch.bfloat16)
    y = torch.randint(0, v, (n,), device=dev, generator=g)
    res = bb.fused_lmhead_loss(h, w, y, bb.FusionConfig(rows_tile, 4096))
    hd, wd = h.double(), w.double()
    logits = hd @ wd.T
    lse = torch.logsumexp(logits, 1)
    loss = lse - logits[torch.arange(n, device=dev), y]
    gm = torch.exp(logits - lse[:, None])
    gm[torch.arange(n, device=dev), y] -= 1
    dh, dw = gm @ wd, gm.T @ hd
    assert float((res.loss.double() - loss).abs().max()) < 2e-3
    assert float(torch.linalg.norm(res.dh.double() - dh) / torch.linalg.norm(dh)) < 1e-2
    assert float(torch.linalg.norm(res.dw.double() - dw) / torch.linalg.norm(dw)) < 1e-2
