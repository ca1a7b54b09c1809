"""Host-side checks of layer.py (no GPU): AttentionParams validation mirrors oracle.py:38-44."""

import numpy as np
import pytest

from paper_2509_19836_b200.layer import AttentionParams


def test_non_square_params_rejected():
    with pytest.raises(ValueError, match="w_q must be 3x3"):
        AttentionParams(dim=3, w_q=np.zeros((3, 2)), w_k=np.zeros((3, 3)), w_v=np.zeros((3, 3)), w_attn=np.zeros((3, 3)))


def test_square_params_accepted():
    p = AttentionParams(dim=2, w_q=np.eye(2), w_k=np.eye(2), w_v=np.eye(2), w_attn=np.eye(2))
    assert p.dim == 2
