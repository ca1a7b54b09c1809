"""Host side of the numerics drop-in (no GPU): the reference's input generator, the
finite-difference utility (oracle.py:157-187) and the burstsim names the package exports."""

import numpy as np
import pytest

import paper_2509_19836_b200 as bb
from golden_data import meta
from paper_2509_19836_b200 import layer as Lyr
from paper_2509_19836_b200 import numerics as F


def test_seeded_random_matrix_golden():
    # pkg/tests/test_numerics.py:175-183 exact values (tests/golden, from burstsim)
    assert np.array_equal(F.seeded_random_matrix(2, 2, 1234), np.array(meta()["seeded_2x2_1234"]))
    assert F.seeded_random_matrix(3, 5, 7).shape == (3, 5)


def test_finite_diff_check_host():
    a = np.array([[1.0, -2.0], [0.5, 3.0]])
    f = lambda x: float(np.sum(x**3))  # noqa: E731
    assert Lyr.finite_diff_check(f, a, 3 * a**2) < 1e-6
    assert Lyr.finite_diff_check(f, a, 3 * a**2 + 1.0) > 0.1
    with pytest.raises(ValueError, match="step size"):
        Lyr.finite_diff_check(f, a, a, h=0.0)
    with pytest.raises(ValueError, match="gradient shape"):
        Lyr.finite_diff_check(f, a, a[:1])
    with pytest.raises(ValueError, match="non-finite"):
        Lyr.finite_diff_check(lambda x: float("inf"), a, a)


def test_reference_numerics_names_exported():
    for name in ("matmul", "row_logsumexp", "row_softmax", "lse_merge", "rowsum_hadamard",
                 "seeded_random_matrix", "naive_lmhead_loss", "finite_diff_check", "numerics"):
        assert hasattr(bb, name), name


@pytest.mark.reference
def test_seeded_random_matrix_equals_reference():
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from burstsim import numerics as R

    for seed in (0, 1, 1234):
        assert np.array_equal(F.seeded_random_matrix(4, 3, seed), R.seeded_random_matrix(4, 3, seed))
