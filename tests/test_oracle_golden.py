"""Pin the CPU oracle (oracle/burst_oracle.py) before trusting it: every function is
checked against golden vectors produced by running the reference itself
(tests/golden/make_golden.py) and against the known-answer tests the reference's
own suite holds (pkg/tests/*.py, cited per test)."""

import math

import numpy as np
import pytest

from golden_data import arrays, meta, oracle_mask, unpack_pairs
from oracle import burst_oracle as O


def test_seeded_matrix_kat():
    # pkg/tests/test_numerics.py:175-183 frozen PCG64 fixture
    assert np.array_equal(O.seeded_random_matrix(2, 2, 1234), np.array(meta()["seeded_2x2_1234"]))


def test_neg_inf_identities():
    # numerics.py:62-69,101-116; pkg/tests/test_distributed.py:64-77
    a = np.array([-np.inf, 1.0, -np.inf])
    b = np.array([2.0, -np.inf, -np.inf])
    assert np.array_equal(O.lse_merge(a, b), np.array([2.0, 1.0, -np.inf]))
    assert np.array_equal(O.exp_gap(np.array([-np.inf]), np.array([-np.inf])), np.array([0.0]))
    s = np.array([[-np.inf, -np.inf], [0.0, 0.0]])
    assert np.array_equal(O.lse_rows(s), np.array([-np.inf, math.log(2.0)]))


def test_layout_kats():
    # pkg/tests/test_partitioning.py:30-50
    assert [list(x) for x in O.shard_ids("zigzag", 8, 2)] == [[1, 2, 7, 8], [3, 4, 5, 6]]
    assert [list(x) for x in O.shard_ids("striped", 8, 2)] == [[1, 3, 5, 7], [2, 4, 6, 8]]
    assert [list(x) for x in O.shard_ids("block_striped", 8, 2, 4)] == [[1, 3, 5, 7], [2, 4, 6, 8]]
    assert list(O.shard_ids("block_striped", 16, 2, 8)[0]) == list(range(1, 17, 2))


def test_layouts_match_reference():
    for rec in meta()["layouts"]:
        got = O.shard_ids(rec["kind"], rec["n"], rec["g"], rec["block_len"])
        assert [list(map(int, x)) for x in got] == rec["ids"], rec["kind"]


def test_local_pairs_and_balance_match_reference():
    for rec in meta()["pairs"]:
        g, n = rec["g"], rec["n"]
        want = unpack_pairs(rec["key"], g, n)
        m = oracle_mask(rec["mask"])
        for idx in range(g * g):
            i, j = idx // g + 1, idx % g + 1
            got = O.local_allowed(rec["kind"], n, g, rec["block_len"], m, i, j)
            assert np.array_equal(got, want[idx]), (rec["key"], i, j)
        per_dev, per_step, total = O.balance_counts(rec["kind"], n, g, rec["block_len"], m)
        assert per_dev == rec["per_device"] and per_step == rec["per_step"] and total == rec["total"]


def test_balance_kats():
    # pkg/tests/test_partitioning.py:142-153
    c = ("causal", None, None, None)
    assert O.balance_counts("contiguous", 8, 2, None, c)[0] == [10, 26]
    assert O.balance_counts("zigzag", 8, 2, None, c)[0] == [18, 18]
    assert O.balance_counts("striped", 8, 2, None, c)[0] == [16, 20]


def test_ring_visit_orders_match_reference():
    for rec in meta()["plans"]:
        if rec["style_req"] != "auto":
            continue
        assert O.ring_visit(rec["nodes"], rec["gpus_per_node"]) == rec["visit"]


def test_comm_closed_forms_match_reference():
    # fabric.py:306-321; pkg/tests/test_fabric.py:98-113
    for rec in meta()["plans"]:
        g = rec["nodes"] * rec["gpus_per_node"]
        for pk, log in rec["logs"].items():
            assert O.comm_elements(pk, rec["n"], rec["d"], g) == log["account"]
    assert O.comm_elements("burst_backward", 16, 4, 4) == 224
    assert abs((3 * 128 + 2) / (4 * 128) - 0.75390625) < 1e-12


def _dist_case(rec):
    n, d = rec["n"], rec["d"]
    s = rec["seeds"]
    q, k, v, do = (O.seeded_random_matrix(n, d, x) for x in s)
    return q, k, v, do


@pytest.mark.parametrize("which", ["burst", "ring"])
def test_ring_passes_match_reference(which):
    A = arrays()
    for rec in meta()["dist"]:
        q, k, v, do = _dist_case(rec)
        visit = O.ring_visit(*rec["topology"])
        res = O.mh_ring_attention(
            q[:, None], k[:, None], v[:, None], do[:, None], (rec["kind"], rec["n"], rec["g"], rec["block_len"]),
            oracle_mask(rec["mask"]), visit, backward=which,
        )
        key = rec["key"]
        pre = "" if which == "burst" else "ring_"
        assert np.max(np.abs(res["o"][:, 0] - A[key + "_o"])) < 1e-12, key
        assert np.max(np.abs(res["lse"][0] - A[key + "_lse"])) < 1e-12, key
        for g_ in ("dq", "dk", "dv"):
            assert np.max(np.abs(res[g_][:, 0] - A[key + f"_{pre}{g_}"])) < 1e-12, (key, g_)


def test_forward_matches_full_materialisation():
    # tests/test_acceptance.py forward tolerance 1e-10 vs oracle.attention_forward
    rec = meta()["dist"][5]
    q, k, v, _ = _dist_case(rec)
    ids = np.arange(1, rec["n"] + 1)
    am = O.allowed(oracle_mask(rec["mask"]), ids, ids)
    o, lse = O.attention_forward(q, k, v, am)
    A = arrays()
    assert np.max(np.abs(o - A[rec["key"] + "_o"])) < 1e-10


def test_globally_masked_row_raises():
    # pkg/tests/test_distributed.py:143-152
    bm = np.array([[0, 0], [1, 1]])
    m = ("block_sparse", None, 4, bm)
    q, k, v = (O.seeded_random_matrix(8, 4, 170 + s) for s in range(3))
    with pytest.raises(ValueError, match="no unmasked key"):
        O.mh_ring_attention(q[:, None], k[:, None], v[:, None], None, ("contiguous", 8, 2, None), m, O.ring_visit(1, 2), backward=None)


def test_lmhead_matches_reference():
    A = arrays()
    for rec in meta()["lmhead"]:
        h = O.seeded_random_matrix(rec["n"], rec["d"], rec["seeds"][0])
        w = O.seeded_random_matrix(rec["v"], rec["d"], rec["seeds"][1])
        y = np.asarray(rec["targets"])
        loss, dh, dw, peak = O.fused_lmhead(h, w, y, rec["bs"], rec["bv"])
        assert np.max(np.abs(loss - A[rec["key"] + "_loss"])) < 1e-12
        assert np.max(np.abs(dh - A[rec["key"] + "_dh"])) < 1e-12
        assert np.max(np.abs(dw - A[rec["key"] + "_dw"])) < 1e-12
        assert peak == rec["peak"]
        nl, _, _ = O.naive_lmhead(h, w, y)
        assert np.max(np.abs(nl - A[rec["key"] + "_naive_loss"])) < 1e-12


def test_lmhead_kats():
    # pkg/tests/test_lmhead.py:25-29: uniform logits give ln 2 and dH = 0
    loss, dh, _, _ = O.fused_lmhead(np.zeros((1, 1)), np.zeros((2, 1)), np.array([0]), 1, 1)
    assert abs(loss[0] - math.log(2)) < 1e-15 and np.allclose(dh, 0)


def test_checkpoint_plan_matches_reference():
    for rec in meta()["ckpt"]:
        m = oracle_mask(rec["mask"])
        stored, rec_pairs, frac, extra = O.checkpoint_plan(rec["policy"], rec["n"], rec["d"], m, rec["split"])
        assert (stored, rec_pairs, extra) == (rec["stored"], rec["recompute_pairs"], rec["extra"])
        assert abs(frac - rec["recompute_fraction"]) < 1e-15
        if rec["policy"] == "sequence_selective":
            assert O.checkpoint_boundary(rec["split"], rec["n"]) == rec["boundary"]


def test_checkpoint_recompute_exact():
    # checkpointing.py:109-172: segment recompute reproduces store-everything grads
    n, d = 32, 8
    q, k, v, do = (O.seeded_random_matrix(n, d, 900 + s) for s in range(4))
    m = ("causal", None, None, None)
    ids = np.arange(1, n + 1)
    am = O.allowed(m, ids, ids)
    o, lse = O.attention_forward(q, k, v, am)
    base = O.attention_backward(q, k, v, o, lse, do, am)
    got, pairs = O.checkpoint_recompute(q, k, v, do, m, np.arange(16, n))
    assert pairs == 16 * 17 // 2  # m(m+1)/2, pkg/tests/test_checkpointing.py:34-61
    for a, b in zip(got, base):
        assert np.max(np.abs(a - b)) < 1e-10


@pytest.mark.parametrize("which", ["burst", "ring"])
def test_cfg4_shaped_case_matches_reference(which):
    """cfg4's structure scaled down (make_cfg4_golden.py): block_striped over 4 devices, a
    sliding-window band AND causal documents as one block_sparse mask, two query heads on one
    K/V head.  The reference ran each query head alone; GQA's dK/dV are their sums."""
    from golden_data import cfg4_golden

    A, n, g, d, lb, mb, hq = cfg4_golden()
    res = O.mh_ring_attention(A["q"], A["k"], A["v"], A["do"], ("block_striped", n, g, lb),
                              ("block_sparse", None, mb, A["block_mask"]), O.ring_visit(1, g), backward=which)
    for h in range(hq):
        assert np.max(np.abs(res["o"][:, h] - A[f"o{h}"])) < 1e-12
        assert np.max(np.abs(res["lse"][h] - A[f"lse{h}"])) < 1e-12
        assert np.max(np.abs(res["dq"][:, h] - A[f"dq{h}"])) < 1e-12
    assert np.max(np.abs(res["dk"][:, 0] - (A["dk0"] + A["dk1"]))) < 1e-12
    assert np.max(np.abs(res["dv"][:, 0] - (A["dv0"] + A["dv1"]))) < 1e-12
    if which == "ring":  # the reference's K/V-circulating pass (head 0 alone) agrees with its burst pass
        r0 = O.mh_ring_attention(A["q"][:, :1], A["k"], A["v"], A["do"][:, :1], ("block_striped", n, g, lb),
                                 ("block_sparse", None, mb, A["block_mask"]), O.ring_visit(1, g), backward="ring")
        for name in ("dq", "dk", "dv"):
            assert np.max(np.abs(r0[name][:, 0] - A[f"ring_{name}0"])) < 1e-12


def test_cfg4_shaped_mask_is_the_bench_construction():
    """The golden's block mask (band AND documents, built inside the generator) is what the
    package's own constructors give: block_mask_from_window AND document_mask (bench.py swa_doc)."""
    from golden_data import cfg4_golden

    from paper_2509_19836_b200.masks import document_mask
    from paper_2509_19836_b200.partitioning import block_mask_from_window

    A, n, *_ = cfg4_golden()
    _, _, _, _, mb, w, doc, _ = (int(x) for x in A["meta"])
    band = block_mask_from_window(n, mb, w).block_mask
    docs = document_mask([doc] * (n // doc), mb).block_mask
    assert np.array_equal(np.logical_and(band, docs).astype(np.int64), A["block_mask"])
