"""Pins for the oracle's thin SVD and recycle-basis selection (oracle.c or_svd;
PAPER.md:519-537 SVD truncation / Schmidt-Eckart-Young, Algorithm 1 :542-559)."""
import numpy as np
import pytest

import oracle


def test_single_column_345():
    U, s, rank, _ = oracle.svd(np.array([[3.0], [4.0], [0.0]]))
    assert rank == 1 and abs(s[0] - 5.0) <= 1e-15
    u = U[:, 0] * np.sign(U[0, 0])
    assert np.allclose(u, [0.6, 0.8, 0.0], rtol=0, atol=1e-15)


def test_orthonormal_input_unit_singular_values(rng):
    Q, _ = np.linalg.qr(rng.standard_normal((20, 4)))
    _, s, rank, _ = oracle.svd(Q)
    assert rank == 4 and np.allclose(s, 1.0, rtol=0, atol=1e-14)


def test_dominant_direction_of_orthogonal_columns():
    X = np.zeros((6, 2))
    X[0, 0] = 1.0          # norm 1
    X[1, 1] = 5.0          # norm 5
    U, s, _, _ = oracle.svd(X)
    assert np.allclose(s, [5.0, 1.0])
    assert abs(abs(U[1, 0]) - 1.0) <= 1e-15


@pytest.mark.parametrize("n,s", [(50, 6), (200, 10), (33, 1)])
def test_vs_numpy_brute_force(rng, n, s):
    X = rng.standard_normal((n, s)) @ np.diag(np.logspace(0, -3, s))
    U, sig, rank, _ = oracle.svd(X)
    sref = np.linalg.svd(X, compute_uv=False)
    assert np.allclose(sig, sref, rtol=1e-13, atol=0)
    assert np.linalg.norm(U.T @ U - np.eye(s)) <= 1e-13
    # left singular vectors: X^T u_i = sigma_i v_i with ||v_i|| = 1, i.e. ||X^T u_i|| = sigma_i
    assert np.allclose(np.linalg.norm(X.T @ U, axis=0), sig, rtol=1e-12)


def test_eckart_young_tail_identity(rng):
    """||X - X_s||_F = sqrt(sum_{i>s} sigma_i^2) for every s (eq. opt_svd)."""
    X = rng.standard_normal((50, 6))
    U, sig, _, _ = oracle.svd(X)
    for s in range(7):
        Xs = U[:, :s] @ (U[:, :s].T @ X)
        assert abs(np.linalg.norm(X - Xs) - np.sqrt(np.sum(sig[s:] ** 2))) <= 1e-12 * np.linalg.norm(X)
    # and beats random rank-s approximations
    for s in (1, 3):
        best = np.linalg.norm(X - U[:, :s] @ (U[:, :s].T @ X))
        for _ in range(50):
            R = rng.standard_normal((50, s)) @ rng.standard_normal((s, 6))
            assert best <= np.linalg.norm(X - R)


def test_known_spectrum_graded(rng):
    """X = P diag(sigma) Q^T with known sigma spanning 1 .. 1e-7: sigma recovered to
    |d sigma_i| <= 1e-15 sigma_1 + 1e-12 sigma_i (one-sided Jacobi with long-double dots)."""
    n, s = 300, 10
    P, _ = np.linalg.qr(rng.standard_normal((n, s)))
    Q, _ = np.linalg.qr(rng.standard_normal((s, s)))
    true = np.logspace(0, -7, s)
    X = P @ np.diag(true) @ Q.T
    _, sig, _, _ = oracle.svd(X)
    assert np.all(np.abs(sig - true) <= 1e-15 * true[0] * 10 + 1e-12 * true)


def test_rank_deficient_window_and_k_eff(rng):
    a, b = rng.standard_normal(40), rng.standard_normal(40)
    X = np.column_stack([a, b, a + b, 2 * a])
    W, sig, k_eff = oracle.recycle_basis(X, 3)
    assert k_eff == 2
    assert np.linalg.norm(W.T @ W - np.eye(2)) <= 1e-12
    # span W subset of span X: projecting W onto X's column space changes nothing
    Qx, _ = np.linalg.qr(np.column_stack([a, b]))
    assert np.linalg.norm(W - Qx @ (Qx.T @ W)) <= 1e-12
    W5, _, k5 = oracle.recycle_basis(X[:, :2], 5)
    assert k5 == 2 and W5.shape == (40, 2)


def test_zero_window():
    U, sig, rank, _ = oracle.svd(np.zeros((5, 3)))
    assert rank == 0 and np.all(sig == 0)


def test_smallest_modes_selection(rng):
    """PAPER.md:673-676 alternative: the k smallest NON-ZERO singular modes.  Known spectrum:
    X = P diag(s) Q^T; the selected span equals span(P[:, rank-k:rank]) and skips zero modes."""
    n, s = 120, 8
    P = np.linalg.qr(rng.standard_normal((n, s)))[0]
    Q = np.linalg.qr(rng.standard_normal((s, s)))[0]
    true = np.array([5.0, 3.0, 2.0, 1.0, 0.5, 0.25, 0.0, 0.0])   # rank 6
    X = P @ np.diag(true) @ Q.T
    W, sig, k_eff = oracle.recycle_basis(X, 2, modes="smallest")
    assert k_eff == 2
    ref = P[:, 4:6]
    assert np.linalg.norm(W @ W.T - ref @ ref.T, 2) <= 1e-10
    Wl, _, _ = oracle.recycle_basis(X, 2)
    assert np.linalg.norm(Wl @ Wl.T - P[:, :2] @ P[:, :2].T, 2) <= 1e-10
    Wall, _, kall = oracle.recycle_basis(X, 10, modes="smallest")
    assert kall == 6                                             # zero modes never selected
