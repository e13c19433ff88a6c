"""CPU: the reduced-order oracle's DEIM (the definition the GPU blocked greedy must reproduce)."""

import numpy as np

from oracle import rom_oracle as R


def test_deim_picks_rows_of_a_permuted_identity():
    perm = np.array([5, 2, 7, 0])
    W = np.zeros((9, 4))
    W[perm, np.arange(4)] = 1.0
    assert np.array_equal(R.deim(W), perm)


def test_deim_interpolation_is_exact_on_the_basis_span():
    rng = np.random.default_rng(1)
    W = rng.standard_normal((200, 12))
    pi = R.deim(W)
    assert len(set(pi.tolist())) == 12
    v = W @ rng.standard_normal(12)
    coef = np.linalg.solve(W[pi], v[pi])
    assert np.max(np.abs(W @ coef - v)) <= 1e-10 * np.max(np.abs(v))


def test_deim_first_row_is_argmax_of_first_column():
    rng = np.random.default_rng(2)
    W = rng.standard_normal((50, 3))
    assert R.deim(W)[0] == int(np.argmax(np.abs(W[:, 0])))
