"""Product host logic (paper_2509_19836_b200: masks, layouts, ring plans, message
accounting, checkpoint plans) must be BIT-EXACT with the reference -- checked
against golden vectors from running burstsim and the reference tests' KATs."""

import numpy as np
import pytest

from golden_data import meta, product_mask, unpack_pairs
from paper_2509_19836_b200 import checkpointing as CK
from paper_2509_19836_b200 import fabric as F
from paper_2509_19836_b200 import masks as M
from paper_2509_19836_b200 import partitioning as P


def test_layout_token_ids_bit_exact():
    for rec in meta()["layouts"]:
        lay = P.ShardLayout(rec["kind"], rec["n"], rec["g"], rec["block_len"])
        got = [list(map(int, x)) for x in P.shard_token_arrays(lay)]
        assert got == rec["ids"]
        assert [list(s.token_ids) for s in P.layout_shards(lay)] == rec["ids"]


@pytest.mark.parametrize(
    "kind,n,g,bl",
    [("contiguous", 10, 4, None), ("striped", 9, 2, None), ("zigzag", 10, 3, None), ("block_striped", 16, 4, 6), ("block_striped", 10, 2, 4)],
)
def test_layout_divisibility_errors(kind, n, g, bl):
    # pkg/tests/test_partitioning.py:52-68
    with pytest.raises(ValueError):
        P.make_layout(kind, n, g, block_len=bl)


def test_local_pair_masks_bit_exact():
    for rec in meta()["pairs"]:
        g, n = rec["g"], rec["n"]
        lay = P.ShardLayout(rec["kind"], n, g, rec["block_len"])
        m = product_mask(rec["mask"])
        want = unpack_pairs(rec["key"], g, n)
        for idx in range(g * g):
            i, j = idx // g + 1, idx % g + 1
            for closed in (True, False):
                assert np.array_equal(P.local_pair_mask(lay, m, i, j, use_closed_form=closed), want[idx])
        rep = P.balance_report(lay, m)
        assert list(rep.per_device_pairs) == rec["per_device"]
        assert [list(r) for r in rep.per_step_pairs] == rec["per_step"]
        assert rep.total_pairs == rec["total"] == P.global_unmasked_pairs(m, n) == rec["global"]
        assert M.unmasked_pair_count(m, n) == rec["global"]


def test_local_pair_set_kats():
    # pkg/tests/test_partitioning.py:80-97
    lay = P.ShardLayout("striped", 8, 2)
    assert P.local_pair_set(lay, M.causal_mask(), 1, 2) == frozenset({(2, 1), (3, 1), (3, 2), (4, 1), (4, 2), (4, 3)})
    z = P.ShardLayout("zigzag", 8, 2)
    assert P.local_pair_set(z, M.causal_mask(), 2, 1) == frozenset((a, b) for a in range(1, 5) for b in (1, 2))
    assert P.local_pair_set(P.ShardLayout("contiguous", 8, 2), M.causal_mask(), 1, 2) == frozenset()
    with pytest.raises(ValueError, match="device indices"):
        P.local_pair_mask(P.ShardLayout("contiguous", 8, 2), M.full_mask(), 0, 1)


def test_balance_kats_and_large_n_counts():
    assert P.balance_report(P.ShardLayout("contiguous", 8, 2), M.causal_mask()).per_device_pairs == (10, 26)
    assert P.balance_report(P.ShardLayout("zigzag", 8, 2), M.causal_mask()).per_device_pairs == (18, 18)
    assert P.balance_report(P.ShardLayout("striped", 8, 2), M.causal_mask()).per_device_pairs == (16, 20)
    # exact pair counts stay cheap at the 1M-token config (no N x N matrix)
    n = 1 << 20
    rep = P.balance_report(P.ShardLayout("zigzag", n, 8), M.causal_mask())
    assert rep.total_pairs == n * (n + 1) // 2 and len(set(rep.per_device_pairs)) == 1
    w = M.sliding_window_mask(32768)
    assert P.global_unmasked_pairs(w, 1 << 19) == 32768 * (1 << 19) - 32768 * 32767 // 2


def test_block_mask_from_window_kats():
    # pkg/tests/test_partitioning.py:194-215
    assert np.array_equal(P.block_mask_from_window(16, 4, 16).block_mask, np.tril(np.ones((4, 4), dtype=np.int64)))
    assert np.array_equal(P.block_mask_from_window(16, 4, 4).block_mask, np.eye(4, dtype=np.int64))
    with pytest.raises(ValueError):
        P.block_mask_from_window(10, 4, 8)
    with pytest.raises(ValueError):
        P.block_mask_from_window(16, 4, 6)


def test_mask_validation_errors():
    with pytest.raises(ValueError):
        M.validate_mask(M.sliding_window_mask(0), 8)
    with pytest.raises(ValueError):
        M.validate_mask(M.block_sparse_mask(np.ones((3, 3)), 4), 8)
    with pytest.raises(ValueError):
        M.block_sparse_mask(np.array([[2]]), 1)
    with pytest.raises(ValueError):
        M.validate_mask(M.MaskSpec("nope"), 8)


def test_document_mask_is_block_sparse():
    dm = M.document_mask([8, 4, 4], block_len=4)
    M.validate_mask(dm, 16)
    ids = np.arange(1, 17)
    a = M.allowed_pairs(dm, ids, ids)
    assert a[0, 0] and not a[0, 4] and a[7, 0] and not a[8, 7] and a[15, 12]


def test_ring_plans_bit_exact():
    for rec in meta()["plans"]:
        topo = F.Topology(rec["nodes"], rec["gpus_per_node"])
        plan = F.build_ring_plan(topo, rec["style_req"])
        assert plan.style == rec["style"]
        assert [list(v) for v in plan.visit] == rec["visit"]
        assert [
            {"label": t.label, "channels": list(t.channels), "receiver": list(t.receiver)} for t in plan.transfers
        ] == rec["transfers"]
        if "intra_rings" in rec:
            dr = F.build_double_ring(topo)
            assert [list(x) for x in dr.intra_rings] == rec["intra_rings"]
            assert [list(x) for x in dr.inter_rings] == rec["inter_rings"]
        g = rec["nodes"] * rec["gpus_per_node"]
        for pk, want in rec["logs"].items():
            log = F.message_log_for(plan, F.step_payload_elements(pk, rec["n"], rec["d"], g))
            assert [log.sent(x) for x in range(1, g + 1)] == want["sent"]
            assert [log.sent(x, "inter") for x in range(1, g + 1)] == want["sent_inter"]
            assert [log.received(x) for x in range(1, g + 1)] == want["received"]
            assert F.account_attention_comm(pk, rec["n"], rec["d"], g) == want["account"]


def test_fabric_kats():
    # pkg/tests/test_fabric.py:98-125
    assert F.account_attention_comm("forward", 16, 4, 4) == 128
    assert F.account_attention_comm("ring_backward", 16, 4, 4) == 256
    assert F.account_attention_comm("burst_backward", 16, 4, 4) == 224
    assert F.step_payload_elements("burst_backward", 16, 4, 4) == 56
    topo = F.Topology(2, 4, lat_intra=3.0, lat_inter=5.0, bw_intra=1e300, bw_inter=1e300)
    assert F.analytic_comm_time("ring", topo, 1.0) == pytest.approx(240.0)
    assert F.analytic_comm_time("double_ring", topo, 1.0) == pytest.approx(128.0)
    assert F.analytic_comm_time("burst", topo, 1.0) == pytest.approx(90.0)
    with pytest.raises(ValueError):
        F.Topology(0, 2)
    with pytest.raises(ValueError):
        F.OverlapSchedule("eager")


def test_validate_timeline_rejects_overlap():
    ev = [F.TimelineEvent(1, "compute", 0.0, 2.0, "a"), F.TimelineEvent(1, "compute", 1.0, 3.0, "b")]
    with pytest.raises(ValueError, match="overlaps"):
        F.validate_timeline(F.Timeline(ev, 3.0))
    ok = [F.TimelineEvent(1, "send_intra", 0.0, 1.0, "s"), F.TimelineEvent(2, "recv", 0.0, 1.0, "recv s")]
    F.validate_timeline(F.Timeline(ok, 1.0))


def test_checkpoint_plans_bit_exact():
    for rec in meta()["ckpt"]:
        pol = CK.CheckpointPolicy(rec["policy"], rec["split"])
        pr = CK.plan(pol, rec["n"], rec["d"], product_mask(rec["mask"]))
        assert pr.stored_elements_per_layer == rec["stored"]
        assert pr.recompute_pairs == rec["recompute_pairs"]
        assert pr.recompute_fraction == rec["recompute_fraction"]
        assert pr.attention_extra_elements == rec["extra"]
        if rec["boundary"] is not None:
            assert pol.boundary(rec["n"]) == rec["boundary"]


def test_checkpoint_dropped_rows_are_a_shard_prefix():
    # the recompute runs the fwd kernel on a row prefix: rows with id <= boundary must be a prefix
    for kind, bl in (("zigzag", None), ("striped", None), ("contiguous", None), ("block_striped", 16)):
        lay = P.ShardLayout(kind, 64, 4, bl)
        b = CK.CheckpointPolicy("sequence_selective", 0.5).boundary(64)
        for ids, p in zip(P.shard_token_arrays(lay), CK._prefix_rows(lay, b)):
            assert np.all(ids[:p] <= b) and np.all(ids[p:] > b)


def test_checkpoint_policy_errors():
    with pytest.raises(ValueError):
        CK.CheckpointPolicy("sequence_selective", 1.0)
    with pytest.raises(ValueError):
        CK.CheckpointPolicy("sequence_selective", 0.3).boundary(16)
    with pytest.raises(ValueError):
        CK.CheckpointPolicy("bogus")


def test_lmhead_models():
    from paper_2509_19836_b200 import lmhead as L

    assert L.memory_footprint(2**20, 128 * 1024, 4096, L.FusionConfig(1024, 4096)) == (2**37, 2**27)
    assert L.tile_working_set(16, 21, 6, L.FusionConfig(4, 7)) == 4 * 6 + 7 * 6 + 16
    for rec in meta()["lmhead"]:
        cfg = L.FusionConfig(rec["bs"], rec["bv"])
        assert list(L.memory_footprint(rec["n"], rec["v"], rec["d"], cfg)) == rec["footprint"]
        assert L.tile_working_set(rec["n"], rec["v"], rec["d"], cfg) == rec["working_set"]
    with pytest.raises(ValueError):
        L.FusionConfig(0, 4)


@pytest.mark.parametrize("kind,n,g,bl", [("contiguous", 64, 4, None), ("zigzag", 64, 4, None), ("zigzag", 64, 1, None),
                                         ("striped", 64, 4, None), ("block_striped", 64, 2, 8)])
def test_shard_rows_numpy_equals_the_reference_gather(kind, n, g, bl):
    """shard_rows on NumPy (distributed.py:118-119): block copies per run of consecutive ids must
    give exactly x[ids - 1], as new arrays (the reference's fancy index never aliases)."""
    from paper_2509_19836_b200.distributed import shard_rows

    layout = P.ShardLayout(kind, n, g, bl)
    for x in (np.random.default_rng(1).standard_normal((n, 3, 5)), np.arange(n * 2, dtype=np.float32).reshape(n, 2)):
        for ids, part in zip(P.shard_token_arrays(layout), shard_rows(layout, x)):
            assert np.array_equal(part, x[np.asarray(ids) - 1]) and part.dtype == x.dtype
            assert not np.shares_memory(part, x)
