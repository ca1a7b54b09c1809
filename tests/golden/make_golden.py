"""Generate golden vectors by running the REFERENCE itself (burstsim, read-only).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.json (integer / structural data) and
tests/golden/golden_fp64.npz (float64 results).  The fixtures travel with the
repo; /root/reference does not exist on the GPU box.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from burstsim import checkpointing, distributed, fabric, lmhead, masks, numerics, oracle, partitioning  # noqa: E402

OUT = Path(__file__).resolve().parent


def mask_cases(n):
    return {
        "full": masks.full_mask(),
        "causal": masks.causal_mask(),
        "window": masks.sliding_window_mask(n // 2 + 1),
        "blockband": partitioning.block_mask_from_window(n, n // 4, n // 2),
    }


def mask_desc(m):
    return {
        "kind": m.kind,
        "window": m.window,
        "block_len": m.block_len,
        "block_mask": None if m.block_mask is None else m.block_mask.tolist(),
    }


def layouts_for(n, g):
    out = [("contiguous", None), ("striped", None)]
    if n % (2 * g) == 0:
        out.append(("zigzag", None))
    if (n // 2) % g == 0:
        out.append(("block_striped", n // 2))
    return out


def main():
    J: dict = {}
    F: dict[str, np.ndarray] = {}

    J["seeded_2x2_1234"] = numerics.seeded_random_matrix(2, 2, 1234).tolist()

    # -- layouts (partitioning.py:85-112)
    J["layouts"] = []
    for n, g in [(8, 1), (8, 2), (16, 2), (16, 4), (32, 4), (64, 8)]:
        for kind, bl in layouts_for(n, g) + [("block_striped", g), ("block_striped", 2 * g)]:
            if kind == "block_striped" and (bl is None or n % bl):
                continue
            lay = partitioning.ShardLayout(kind, n, g, block_len=bl)
            J["layouts"].append(
                {"kind": kind, "n": n, "g": g, "block_len": bl, "ids": [list(map(int, t)) for t in partitioning.shard_token_arrays(lay)]}
            )

    # -- local pair masks + balance (partitioning.py:120-225)
    J["pairs"] = []
    for n, g in [(16, 2), (16, 4), (32, 4)]:
        for kind, bl in layouts_for(n, g):
            lay = partitioning.ShardLayout(kind, n, g, block_len=bl)
            for mname, m in mask_cases(n).items():
                key = f"pairs_{kind}_{n}_{g}_{mname}"
                stack = np.stack(
                    [partitioning.local_pair_mask(lay, m, i, j) for i in range(1, g + 1) for j in range(1, g + 1)]
                )
                F[key] = np.packbits(stack.astype(np.uint8), axis=-1)
                rep = partitioning.balance_report(lay, m)
                J["pairs"].append(
                    {
                        "key": key, "kind": kind, "n": n, "g": g, "block_len": bl, "mask": mask_desc(m), "mask_name": mname,
                        "per_device": list(rep.per_device_pairs), "per_step": [list(r) for r in rep.per_step_pairs],
                        "total": rep.total_pairs, "global": partitioning.global_unmasked_pairs(m, n),
                    }
                )

    # -- ring plans + message logs (fabric.py:102-327)
    J["plans"] = []
    for r, m in [(1, 1), (1, 2), (1, 4), (1, 8), (2, 2), (2, 4), (4, 2), (2, 1)]:
        topo = fabric.Topology(r, m)
        for style in ("auto", "flat", "double"):
            plan = fabric.build_ring_plan(topo, style)
            rec = {
                "nodes": r, "gpus_per_node": m, "style_req": style, "style": plan.style,
                "visit": [list(v) for v in plan.visit],
                "transfers": [{"label": t.label, "channels": list(t.channels), "receiver": list(t.receiver)} for t in plan.transfers],
            }
            if r * m > 1:
                dr = fabric.build_double_ring(topo)
                rec["intra_rings"] = [list(x) for x in dr.intra_rings]
                rec["inter_rings"] = [list(x) for x in dr.inter_rings]
            n, d = 16 * r * m, 4
            logs = {}
            for pk in fabric.PASS_KINDS:
                log = fabric.message_log_for(plan, fabric.step_payload_elements(pk, n, d, r * m))
                logs[pk] = {
                    "sent": [log.sent(x) for x in range(1, r * m + 1)],
                    "sent_inter": [log.sent(x, "inter") for x in range(1, r * m + 1)],
                    "received": [log.received(x) for x in range(1, r * m + 1)],
                    "account": fabric.account_attention_comm(pk, n, d, r * m),
                }
            rec["n"], rec["d"], rec["logs"] = n, d, logs
            J["plans"].append(rec)

    # -- distributed passes (distributed.py:151-299), single head, fp64
    J["dist"] = []
    cid = 0
    for n, d, g in [(16, 4, 1), (16, 8, 2), (16, 4, 4), (32, 8, 4), (64, 16, 8), (32, 16, 2)]:
        q, k, v = (numerics.seeded_random_matrix(n, d, 1000 + cid * 10 + s) for s in range(3))
        do = numerics.seeded_random_matrix(n, d, 1000 + cid * 10 + 3)
        cid += 1
        for kind, bl in layouts_for(n, g):
            lay = partitioning.ShardLayout(kind, n, g, block_len=bl)
            for mname, m in mask_cases(n).items():
                for topo_shape in ([(1, g)] + ([(2, g // 2)] if g >= 4 else [])):
                    topo = fabric.Topology(*topo_shape)
                    st = distributed.make_device_states(lay, q, k, v)
                    distributed.distributed_forward(st, lay, m, topo)
                    do_sh = distributed.shard_rows(lay, do)
                    distributed.burst_backward(st, do_sh, lay, m, topo)
                    st2 = distributed.make_device_states(lay, q, k, v)
                    distributed.distributed_forward(st2, lay, m, topo)
                    distributed.ring_backward(st2, do_sh, lay, m, topo)
                    key = f"dist_{n}_{d}_{g}_{kind}_{mname}_{topo_shape[0]}x{topo_shape[1]}"
                    gr = lambda arrs: distributed.gather_rows(lay, arrs)  # noqa: E731
                    F[key + "_o"] = gr([s.o for s in st])
                    F[key + "_lse"] = gr([s.lse for s in st])
                    F[key + "_dq"] = gr([s.dq for s in st])
                    F[key + "_dk"] = gr([s.dk for s in st])
                    F[key + "_dv"] = gr([s.dv for s in st])
                    F[key + "_delta"] = gr([s.d_vec for s in st])
                    F[key + "_ring_dq"] = gr([s.dq for s in st2])
                    F[key + "_ring_dk"] = gr([s.dk for s in st2])
                    F[key + "_ring_dv"] = gr([s.dv for s in st2])
                    J["dist"].append(
                        {"key": key, "n": n, "d": d, "g": g, "kind": kind, "block_len": bl, "mask": mask_desc(m),
                         "topology": list(topo_shape), "seeds": [1000 + (cid - 1) * 10 + s for s in range(4)]}
                    )

    # -- LM head (lmhead.py:41-116; oracle.py:129-154)
    J["lmhead"] = []
    for n, v, d, bs, bv in [(6, 11, 4, 2, 3), (16, 33, 8, 3, 5), (64, 257, 16, 8, 32), (12, 29, 5, 4, 7), (40, 100, 8, 40, 100)]:
        h = numerics.seeded_random_matrix(n, d, 500 + n)
        w = numerics.seeded_random_matrix(v, d, 501 + n)
        y = np.random.default_rng(502 + n).integers(0, v, size=n)
        res = lmhead.fused_lmhead_loss(h, w, y, lmhead.FusionConfig(bs, bv))
        nav = oracle.naive_lmhead_loss(h, w, y)
        key = f"lm_{n}_{v}_{d}_{bs}_{bv}"
        F[key + "_loss"], F[key + "_dh"], F[key + "_dw"] = res.loss, res.dh, res.dw
        F[key + "_naive_loss"] = nav.loss
        J["lmhead"].append(
            {"key": key, "n": n, "v": v, "d": d, "bs": bs, "bv": bv, "seeds": [500 + n, 501 + n, 502 + n],
             "targets": list(map(int, y)), "peak": res.peak_aux_elements,
             "footprint": list(lmhead.memory_footprint(n, v, d, lmhead.FusionConfig(bs, bv))),
             "working_set": lmhead.tile_working_set(n, v, d, lmhead.FusionConfig(bs, bv))}
        )

    # -- checkpointing (checkpointing.py:36-172)
    J["ckpt"] = []
    for n, d in [(16, 4), (32, 8), (64, 4)]:
        for mname, m in mask_cases(n).items():
            for pol in (
                checkpointing.CheckpointPolicy("full_recompute"),
                checkpointing.CheckpointPolicy("selective_pp"),
                checkpointing.CheckpointPolicy("sequence_selective", 0.5),
                checkpointing.CheckpointPolicy("sequence_selective", 0.25),
            ):
                pr = checkpointing.plan(pol, n, d, m)
                toy = checkpointing.execute_toy(pol, n, d, m, seed=77)
                J["ckpt"].append(
                    {"n": n, "d": d, "mask": mask_desc(m), "mask_name": mname, "policy": pol.kind, "split": pol.split_fraction,
                     "stored": pr.stored_elements_per_layer, "recompute_pairs": pr.recompute_pairs,
                     "recompute_fraction": pr.recompute_fraction, "extra": pr.attention_extra_elements,
                     "toy_recomputed_pairs": toy.recomputed_pairs, "toy_matches": toy.matches_baseline,
                     "boundary": pol.boundary(n) if pol.kind == "sequence_selective" else None}
                )

    (OUT / "golden.json").write_text(json.dumps(J, separators=(",", ":")))
    np.savez_compressed(OUT / "golden_fp64.npz", **F)
    print(f"wrote {len(F)} arrays, json {len(json.dumps(J)) // 1024} KB")


if __name__ == "__main__":
    main()
