"""One GPU: attn_bwd_step over kv-head halves equals the full step (every (i, j) of a G=4 zigzag
causal ring, GQA 4q/2kv); guards the kv_head range of bb_attn_bwd_step."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_19836_b200 import kernels as K, masks as M
from paper_2509_19836_b200.partitioning import ShardLayout

dev = torch.device("cuda", 0)
for hq, hkv in ((4, 2), (4, 4), (8, 2)):
    G, n, d = 4, 4096, 128
    lay = ShardLayout("zigzag", n, G)
    dm = K.device_mask(M.causal_mask(), dev)
    g = torch.Generator(device=dev).manual_seed(0)
    r = lambda h: (torch.rand(n // G, h, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    q, k, v, do = r(hq), r(hkv), r(hkv), r(hq)
    lse = torch.rand(hq, n // G, device=dev) + 5
    delta = torch.rand(hq, n // G, device=dev)
    worst = 0.0
    for i in range(G):
        for j in range(G):
            outs = []
            for split in (False, True):
                dq = torch.zeros(n // G, hq, d, device=dev); dk = torch.zeros(n // G, hkv, d, device=dev); dv = torch.zeros_like(dk)
                heads = [(0, hkv // 2), (hkv // 2, hkv)] if split else [None]
                for h in heads:
                    K.attn_bwd_step(q, k, v, do, lse, delta, dq, dk, dv, lay, dm, i + 1, j + 1, 0.088, kv_heads=h)
                torch.cuda.synchronize(); outs.append((dq, dk, dv))

            for a, b in zip(*outs):
                worst = max(worst, float((a - b).abs().max()) / (float(b.abs().max()) + 1e-30))
    print(f"hq={hq} hkv={hkv}: max rel diff split vs full {worst:.2e}", flush=True)
    assert worst < 1e-5
print("OK")
