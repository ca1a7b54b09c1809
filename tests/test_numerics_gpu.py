"""burstsim.numerics / oracle.naive_lmhead_loss on the device (paper_2509_19836_b200.numerics,
csrc/bb_numerics.cu) against the CPU oracle and the reference's golden vectors, in float64.

Cases follow pkg/tests/test_numerics.py: the -inf identities are exact (lse_merge(-inf, x) == x,
exp_gap(-inf, .) == 0, all -inf rows give -inf), fully masked rows are errors for row_softmax,
shape mismatches raise ValueError.  Values agree with NumPy to a few ulps (reduction order
differs from einsum's: tolerance 1e-13 relative, stated per test); the LM head matches the
reference's own outputs (tests/golden, produced by running burstsim) to 1e-12."""

import math

import numpy as np
import pytest
import torch

from golden_data import arrays, meta
from oracle import burst_oracle as O
from paper_2509_19836_b200 import _native
from paper_2509_19836_b200 import layer as Lyr
from paper_2509_19836_b200 import numerics as F

pytestmark = pytest.mark.gpu
INF = math.inf


def _close(a, b, rtol=1e-13):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    assert np.array_equal(np.isneginf(a), np.isneginf(b))
    fin = np.isfinite(b)
    assert np.all(np.abs(a[fin] - b[fin]) <= rtol * (1 + np.abs(b[fin])))


@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (7, 5, 3), (64, 64, 64), (130, 257, 67), (300, 1, 200)])
def test_matmul_matches_numpy(cuda, m, k, n):
    a, b = O.seeded_random_matrix(m, k, 1), O.seeded_random_matrix(k, n, 2)
    launches = _native.launch_count()
    _close(F.matmul(a, b), O.mm(a, b), 1e-13)
    assert _native.launch_count() > launches


def test_matmul_transposed_views_and_device_tensors(cuda):
    a, b = O.seeded_random_matrix(40, 33, 3), O.seeded_random_matrix(21, 33, 4)
    ta, tb = torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda)
    out = F.matmul(ta, tb.t())  # B^T as a stride swap
    assert isinstance(out, torch.Tensor) and out.is_cuda
    _close(out.cpu().numpy(), a @ b.T, 1e-13)
    _close(F.matmul(ta.t(), ta).cpu().numpy(), a.T @ a, 1e-13)


def test_matmul_deterministic_and_errors(cuda):
    a, b = O.seeded_random_matrix(100, 90, 5), O.seeded_random_matrix(90, 80, 6)
    assert np.array_equal(F.matmul(a, b), F.matmul(a, b))
    with pytest.raises(ValueError, match="matmul shape mismatch"):
        F.matmul(a, a)
    with pytest.raises(ValueError, match="2-dimensional"):
        F.matmul(np.zeros(3), b)
    assert F.matmul(np.zeros((3, 0)), np.zeros((0, 2))).tolist() == [[0.0, 0.0]] * 3


def test_row_logsumexp_and_inf_rows(cuda):
    s = O.seeded_random_matrix(37, 300, 7) * 30
    s[3] = -INF
    s[5, ::2] = -INF
    _close(F.row_logsumexp(s), O.lse_rows(s))
    assert F.row_logsumexp(s)[3] == -INF
    # numerics.py:48-59: single-element rows are exact
    assert F.row_logsumexp(np.array([[2.5]]))[0] == 2.5
    with pytest.raises(ValueError, match="nonempty"):
        F.row_logsumexp(np.zeros((0, 3)))


def test_lse_merge_identities(cuda):
    a = np.array([-INF, -INF, 1.0, 2.0, 0.0, -3.5, 700.0])
    b = np.array([-INF, 4.0, -INF, 2.0, 1e-3, 10.0, -700.0])
    out = F.lse_merge(a, b)
    ref = np.logaddexp(a, b)
    assert out[0] == -INF and out[1] == 4.0 and out[2] == 1.0  # -inf is the identity, exactly
    _close(out, ref, 1e-15)
    with pytest.raises(ValueError, match="length mismatch"):
        F.lse_merge(a, b[:3])


def test_exp_shifted_exp_gap_rowsum(cuda):
    s = O.seeded_random_matrix(9, 17, 8)
    lse = O.lse_rows(s)
    lse[4] = -INF
    out = F.exp_shifted(s, lse)
    assert np.all(out[4] == 0.0)
    _close(out, O.exp_shifted(s, lse), 1e-14)
    a = np.array([-INF, 0.0, -2.0, 3.0])
    b = np.array([5.0, -INF, -1.0, 3.0])
    g = F.exp_gap(a, b)
    assert g[0] == 0.0 and g[1] == INF and g[3] == 1.0
    _close(g[2:], O.exp_gap(a, b)[2:], 1e-15)
    x, y = O.seeded_random_matrix(50, 129, 9), O.seeded_random_matrix(50, 129, 10)
    _close(F.rowsum_hadamard(x, y), O.rowsum_hadamard(x, y), 1e-13)
    with pytest.raises(ValueError, match="shape mismatch"):
        F.rowsum_hadamard(x, y[:, :3])


def test_row_softmax(cuda):
    s = O.seeded_random_matrix(6, 11, 11)
    p = F.row_softmax(s)
    _close(p.sum(axis=1), np.ones(6), 1e-14)
    s[2] = -INF
    with pytest.raises(ValueError, match="row 2 is fully masked"):
        F.row_softmax(s)


def test_naive_lmhead_matches_reference_golden(cuda):
    A = arrays()
    for rec in meta()["lmhead"]:
        h = O.seeded_random_matrix(rec["n"], rec["d"], rec["seeds"][0])
        w = O.seeded_random_matrix(rec["v"], rec["d"], rec["seeds"][1])
        y = np.asarray(rec["targets"])
        res = Lyr.naive_lmhead_loss(h, w, y)
        assert np.max(np.abs(res.loss - A[rec["key"] + "_naive_loss"])) < 1e-12
        # fused and naive heads agree in the reference to 1e-10 (pkg/tests/test_lmhead.py)
        assert np.max(np.abs(res.dh - A[rec["key"] + "_dh"])) < 1e-10
        assert np.max(np.abs(res.dw - A[rec["key"] + "_dw"])) < 1e-10


def test_naive_lmhead_kats_and_errors(cuda):
    # pkg/tests/test_lmhead.py:25-29: uniform logits give ln 2 and dH = 0
    res = Lyr.naive_lmhead_loss(np.zeros((1, 1)), np.zeros((2, 1)), np.array([0]))
    assert abs(res.loss[0] - math.log(2)) < 1e-15 and np.all(res.dh == 0)
    with pytest.raises(ValueError, match="outside"):
        Lyr.naive_lmhead_loss(np.zeros((2, 3)), np.zeros((4, 3)), np.array([0, 4]))
    with pytest.raises(ValueError, match="columns"):
        Lyr.naive_lmhead_loss(np.zeros((2, 3)), np.zeros((4, 2)), np.array([0, 1]))


def test_naive_lmhead_finite_difference(cuda):
    h, w = O.seeded_random_matrix(3, 4, 20), O.seeded_random_matrix(5, 4, 21)
    y = np.array([1, 4, 0])
    res = Lyr.naive_lmhead_loss(h, w, y)
    assert Lyr.finite_diff_check(lambda x: Lyr.naive_lmhead_loss(x, w, y).loss.sum(), h, res.dh) < 1e-5
    assert Lyr.finite_diff_check(lambda x: Lyr.naive_lmhead_loss(h, x, y).loss.sum(), w, res.dw) < 1e-5


def test_exp_shifted_many_rows(cuda):
    # more rows than a CUDA grid's y extent: the kernel walks rows x cols flat
    s = O.seeded_random_matrix(70001, 3, 12)
    lse = O.lse_rows(s)
    lse[70000] = -INF
    out = F.exp_shifted(s, lse)
    assert np.all(out[70000] == 0.0)
    _close(out, O.exp_shifted(s, lse), 1e-14)


def test_masked_scores_matches_reference_algorithm(cuda):
    # oracle.py:66-75: S = Q K^T / sqrt(d), masked entries exactly -inf
    from paper_2509_19836_b200.masks import causal_mask, dense_mask, sliding_window_mask

    q, k = O.seeded_random_matrix(12, 5, 30), O.seeded_random_matrix(12, 5, 31)
    for mask in (causal_mask(), sliding_window_mask(3)):
        s = Lyr.masked_scores(q, k, mask)
        allowed = dense_mask(mask, 12, 12)
        want = np.where(allowed, O.mm(q, k.T) / np.sqrt(5), -INF)
        _close(s, want, 1e-14)
    with pytest.raises(ValueError, match="dim"):
        Lyr.masked_scores(q, k[:, :3], causal_mask())
