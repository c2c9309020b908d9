"""Pins for the oracle's SSOR preconditioner and right-preconditioned solves (oracle.c ssor_apply,
or_ssor, or_solve_pc).

SSOR ("Symmetric Successive Over-Relaxation (SSOR) preconditioner"), textbook form in a row
order: M = (D + wL) D^{-1} (D + wU) / (w(2-w)).  Right preconditioning ("A M y = b,
x = M^{-1} y"; R18): search space x_c + [span W] + M^{-1} K_j(op A M^{-1}, v).
"""
import numpy as np
import pytest

import oracle
from bruteforce import random_nonsym, restarted_minres, restarted_oblique, ssor_matrix


def _grid5(N, rng, conv=0.3):
    """5-point convection-diffusion-like operator on an N x N grid (dense), diagonally dominant."""
    n = N * N
    D = np.zeros((n, n))
    for i in range(N):
        for j in range(N):
            r = i * N + j
            D[r, r] = 4.0 + 0.5 + rng.random()
            for di, dj, s in ((-1, 0, 1 + conv), (1, 0, 1 - conv), (0, -1, 1 + conv), (0, 1, 1 - conv)):
                ii, jj = i + di, j + dj
                if 0 <= ii < N and 0 <= jj < N:
                    D[r, ii * N + jj] = -s
    return D


def _red_black(N):
    return np.array([(i + j) % 2 for i in range(N) for j in range(N)])


@pytest.mark.parametrize("omega", [1.0, 0.7, 1.5])
def test_ssor_equals_inverse_of_assembled_matrix(rng, omega):
    n = 30
    D = random_nonsym(n, rng, shift=3.0)
    order = rng.permutation(n).astype(np.int32)
    z = rng.standard_normal(n)
    got = oracle.ssor(oracle.Matrix.from_dense(D), order, omega, z)
    ref = np.linalg.solve(ssor_matrix(D, order, omega), z)
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


def test_diagonal_closed_form(rng):
    """A = D (no off-diagonal entries): M = D / (w(2-w)) ... at w = 1, M^{-1} z = z / d."""
    d = rng.random(12) + 0.5
    A = oracle.Matrix.from_dense(np.diag(d))
    z = rng.standard_normal(12)
    order = np.arange(12, dtype=np.int32)
    assert np.allclose(oracle.ssor(A, order, 1.0, z), z / d, rtol=1e-15, atol=0)
    assert np.allclose(oracle.ssor(A, order, 0.5, z), 0.75 * z / d, rtol=1e-15, atol=0)


def test_symmetric_matrix_gives_symmetric_preconditioner(rng):
    n = 25
    G = rng.standard_normal((n, n))
    S = G + G.T + 2 * n * np.eye(n)
    A = oracle.Matrix.from_dense(S)
    order = rng.permutation(n).astype(np.int32)
    z1, z2 = rng.standard_normal(n), rng.standard_normal(n)
    a = z2 @ oracle.ssor(A, order, 1.3, z1)
    b = z1 @ oracle.ssor(A, order, 1.3, z2)
    assert abs(a - b) <= 1e-13 * max(abs(a), 1.0)


def test_lower_triangular_in_order_forward_sweep_is_exact(rng):
    """A lower triangular in the processing order and w = 1: U = 0, so M = (D + L) and M^{-1} z
    solves A y = z exactly."""
    n = 15
    order = rng.permutation(n).astype(np.int32)
    Lp = np.tril(rng.standard_normal((n, n)), -1) + np.diag(rng.random(n) + 1.0)
    Dm = np.empty_like(Lp)
    Dm[np.ix_(order, order)] = Lp
    z = rng.standard_normal(n)
    y = oracle.ssor(oracle.Matrix.from_dense(Dm), order, 1.0, z)
    assert np.linalg.norm(Dm @ y - z) <= 1e-13 * np.linalg.norm(z)


def test_multicolour_order_is_a_valid_ssor_order(rng):
    """Red-black order on a 5-point grid: the result equals the assembled SSOR of that order, and
    rows inside one colour do not couple (the order inside a colour does not matter)."""
    N = 7
    D = _grid5(N, rng)
    col = _red_black(N)
    o1 = oracle.ssor_order(col)
    o2 = np.concatenate([np.flatnonzero(col == 0)[::-1], np.flatnonzero(col == 1)[::-1]]).astype(np.int32)
    z = rng.standard_normal(N * N)
    A = oracle.Matrix.from_dense(D)
    a, b = oracle.ssor(A, o1, 1.0, z), oracle.ssor(A, o2, 1.0, z)
    assert np.linalg.norm(a - b) <= 1e-14 * np.linalg.norm(a)
    assert np.linalg.norm(a - np.linalg.solve(ssor_matrix(D, o1, 1.0), z)) <= 1e-13 * np.linalg.norm(a)


@pytest.mark.parametrize("variant", ["plain", "augment", "deflate"])
def test_right_preconditioned_matches_brute_force(rng, variant):
    N = 6
    D = _grid5(N, rng, conv=0.6)
    n = N * N
    W = np.linalg.qr(rng.standard_normal((n, 3)))[0]
    b = rng.standard_normal(n)
    order = oracle.ssor_order(_red_black(N))
    Minv = np.linalg.inv(ssor_matrix(D, order, 1.0))
    r = oracle.solve(oracle.Matrix.from_dense(D), b, m=5, variant=variant, W=W, tol=1e-10,
                     max_iters=300, precond=(order, 1.0))
    xb, itb, hb = restarted_minres(D, b, 5, variant=variant, W=W, tol=1e-10, max_iters=300, Minv=Minv)
    assert r["converged"] and r["iterations"] == itb
    kk = min(len(hb), len(r["history"]))
    assert np.allclose(r["history"][:kk], hb[:kk], rtol=1e-7, atol=1e-13)
    assert np.linalg.norm(r["x"] - xb) <= 1e-8 * np.linalg.norm(xb)


def test_right_preconditioned_oblique_matches_brute_force(rng):
    N = 6
    D = _grid5(N, rng, conv=0.6)
    n = N * N
    W = np.linalg.qr(rng.standard_normal((n, 3)))[0]
    b = rng.standard_normal(n)
    order = oracle.ssor_order(_red_black(N))
    Minv = np.linalg.inv(ssor_matrix(D, order, 1.2))
    r = oracle.solve(oracle.Matrix.from_dense(D), b, m=5, variant="oblique", W=W, tol=1e-10,
                     max_iters=300, precond=(order, 1.2))
    xb, itb, hb = restarted_oblique(D, b, 5, W, tol=1e-10, max_iters=300, Minv=Minv)
    assert r["converged"] and r["iterations"] == itb
    assert np.linalg.norm(r["x"] - xb) <= 1e-8 * np.linalg.norm(xb)


def test_exact_preconditioner_converges_in_one_step(rng):
    """A lower triangular in the order, w = 1: M = A, so A M^{-1} = I and GMRES stops after one
    step with the exact solution (right preconditioning keeps the TRUE residual)."""
    n = 20
    order = rng.permutation(n).astype(np.int32)
    Lp = np.tril(rng.standard_normal((n, n)) * 0.3, -1) + np.diag(rng.random(n) + 1.0)
    Dm = np.empty_like(Lp)
    Dm[np.ix_(order, order)] = Lp
    b = rng.standard_normal(n)
    r = oracle.solve(oracle.Matrix.from_dense(Dm), b, m=10, tol=1e-12, precond=(order, 1.0))
    assert r["iterations"] == 1 and r["converged"]
    assert np.linalg.norm(r["x"] - np.linalg.solve(Dm, b)) <= 1e-12 * np.linalg.norm(r["x"])


def test_preconditioning_reduces_iterations_on_grid(rng):
    N = 12
    D = _grid5(N, rng, conv=0.5)
    b = rng.standard_normal(N * N)
    A = oracle.Matrix.from_dense(D)
    order = oracle.ssor_order(_red_black(N))
    p0 = oracle.solve(A, b, m=10, tol=1e-10)
    p1 = oracle.solve(A, b, m=10, tol=1e-10, precond=(order, 1.0))
    assert p1["converged"] and p1["iterations"] < p0["iterations"]
    assert np.linalg.norm(b - D @ p1["x"]) <= 1e-10 * np.linalg.norm(b)


def test_zero_diagonal_reported():
    D = np.array([[0.0, 1.0], [1.0, 2.0]])
    with pytest.raises(np.linalg.LinAlgError):
        oracle.ssor(oracle.Matrix.from_dense(D), np.array([0, 1], np.int32), 1.0, np.ones(2))
