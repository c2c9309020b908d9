"""Pins for the oracle's Galerkin/oblique variants (oracle.c solve_oblique, or_obproj; SURVEY §8(f)
NEXT #1).

M_D = I - A W E^{-1} W^T, E = W^T A W          (eq. left_deflation)
rows 5 / 2 of Table 1: Krylov operator M_D A, initial vector M_D r_0 / r_0
start x_0 = W E^{-1} W^T b                        (eq. projection_t_s :419)
rows 2 and 5 coincide without preconditioning     (eq. equivalence_oblique)
"""
import numpy as np
import pytest

import oracle
from bruteforce import oblique_projector, random_nonsym, restarted_oblique


def _orthonormal(n, k, rng):
    return np.linalg.qr(rng.standard_normal((n, k)))[0]


def test_projector_defining_properties(rng):
    """A projector is fixed by its range and null space: M_D A W = 0 (null space >= range(AW),
    P:239 'by construction M_D A V_s = 0'), W^T M_D = 0 (range <= W-perp), M_D^2 = M_D and
    rank n - k pin or_obproj to the unique oblique projector onto W-perp along range(AW)."""
    n, k = 40, 4
    D = random_nonsym(n, rng)
    W = _orthonormal(n, k, rng)
    A = oracle.Matrix.from_dense(D)
    assert np.linalg.norm(oracle.obproj(A, W, D @ W)) <= 1e-12 * np.linalg.norm(D)
    Mfull = oracle.obproj(A, W, np.eye(n))
    assert np.linalg.norm(W.T @ Mfull) <= 1e-12 * np.linalg.norm(Mfull)
    assert np.linalg.norm(Mfull @ Mfull - Mfull) <= 1e-12 * np.linalg.norm(Mfull)
    assert np.linalg.matrix_rank(Mfull, tol=1e-8) == n - k
    # and the literal formula of P:233 (written out independently in bruteforce.py)
    assert np.linalg.norm(Mfull - oblique_projector(D, W)) <= 1e-11 * np.linalg.norm(Mfull)


@pytest.mark.parametrize("row2", [False, True])
@pytest.mark.parametrize("m,k", [(5, 3), (9, 1), (4, 6)])
def test_matches_brute_force_explicit_space(rng, row2, m, k):
    """Every step's residual = explicit lstsq minimum of ||M_D r_c - M_D A z|| over the monomial
    Krylov space of M_D A (restarts included); same iterates."""
    n = 36
    D = random_nonsym(n, rng, shift=1.4)
    W = _orthonormal(n, k, rng)
    b = rng.standard_normal(n)
    var = "oblique_aug" if row2 else "oblique"
    r = oracle.solve(oracle.Matrix.from_dense(D), b, m=m, variant=var, W=W, tol=1e-9, max_iters=400)
    xb, itb, hb = restarted_oblique(D, b, m, W, tol=1e-9, max_iters=400, row2=row2)
    assert r["converged"]
    assert r["iterations"] == itb
    kk = min(len(hb), len(r["history"]))
    assert np.allclose(r["history"][:kk], hb[:kk], rtol=1e-7, atol=1e-12)
    assert np.linalg.norm(r["x"] - xb) <= 1e-7 * np.linalg.norm(xb)


def test_minimised_residual_is_true_residual_after_galerkin_correction(rng):
    """After j steps the returned x (Galerkin-corrected) has TRUE residual ||b - A x|| equal to
    the minimised ||M_D (r_0 - A z)|| (the last history entry): M_D r = r - A W E^{-1} W^T r."""
    n, k = 50, 3
    D = random_nonsym(n, rng, shift=1.2)
    W = _orthonormal(n, k, rng)
    b = rng.standard_normal(n)
    for j in (1, 2, 5, 8):
        r = oracle.solve(oracle.Matrix.from_dense(D), b, m=20, variant="oblique", W=W, tol=1e-14, max_iters=j)
        assert r["iterations"] == j
        true = np.linalg.norm(b - D @ r["x"]) / np.linalg.norm(b)
        assert abs(true - r["history"][-1]) <= 1e-10 * max(true, 1e-3)
        assert abs(r["rel_residual"] - true) <= 1e-12


def test_rows_2_and_5_equivalent(rng):
    """eq. equivalence_oblique: with the Galerkin start, M_D r_0 = r_0, so the augmented and
    deflated oblique methods give the same iterates (restarts included, m = 6)."""
    n, k = 80, 5
    D = random_nonsym(n, rng, shift=1.1)
    W = _orthonormal(n, k, rng)
    b = rng.standard_normal(n)
    A = oracle.Matrix.from_dense(D)
    p = oracle.solve(A, b, m=6, variant="oblique", W=W, tol=1e-10, max_iters=500)
    q = oracle.solve(A, b, m=6, variant="oblique_aug", W=W, tol=1e-10, max_iters=500)
    assert p["converged"] and q["converged"]
    assert p["iterations"] == q["iterations"] and p["cycles"] > 1
    assert np.allclose(p["history"], q["history"], rtol=1e-8, atol=1e-13)
    assert np.linalg.norm(p["x"] - q["x"]) <= 1e-9 * np.linalg.norm(p["x"])


def test_rhs_in_image_of_recycle_space(rng):
    """b = A W c  =>  the Galerkin start W E^{-1} W^T b = W c solves it: 0 iterations."""
    n, k = 30, 4
    D = random_nonsym(n, rng)
    W = _orthonormal(n, k, rng)
    c = rng.standard_normal(k)
    r = oracle.solve(oracle.Matrix.from_dense(D), D @ W @ c, m=10, variant="oblique", W=W)
    assert r["iterations"] == 0 and r["converged"]
    assert np.linalg.norm(r["x"] - W @ c) <= 1e-12 * np.linalg.norm(c)


def test_dense_solution_and_final_orthogonality(rng):
    """Converges to the LU solution; on return W^T (b - A x) = 0 (the final Galerkin/oblique
    correction, eq. projection_guess 'V_s^T r_0 = 0')."""
    n, k = 60, 5
    D = random_nonsym(n, rng, shift=1.3)
    W = _orthonormal(n, k, rng)
    b = rng.standard_normal(n)
    r = oracle.solve(oracle.Matrix.from_dense(D), b, m=8, variant="oblique", W=W, tol=1e-11, max_iters=2000)
    xs = np.linalg.solve(D, b)
    assert r["converged"]
    assert np.linalg.norm(r["x"] - xs) <= 1e-8 * np.linalg.norm(xs)
    assert np.linalg.norm(W.T @ (b - D @ r["x"])) <= 1e-13 * np.linalg.norm(b)


def test_singular_restriction_reported():
    """E = W^T A W singular (A skew on span W): reported, not silently used."""
    D = np.eye(4) * 2.0
    D[0, 0] = D[1, 1] = 0.0
    D[0, 1], D[1, 0] = 1.0, -1.0
    W = np.zeros((4, 1))
    W[0, 0] = 1.0
    with pytest.raises(np.linalg.LinAlgError):
        oracle.solve(oracle.Matrix.from_dense(D), np.ones(4), m=4, variant="oblique", W=W)


def test_empty_recycle_space_is_plain(rng):
    n = 30
    D = random_nonsym(n, rng, shift=1.5)
    b = rng.standard_normal(n)
    A = oracle.Matrix.from_dense(D)
    p = oracle.solve(A, b, m=6, variant="plain")
    q = oracle.solve(A, b, m=6, variant="oblique", W=None)
    assert p["iterations"] == q["iterations"] and np.array_equal(p["x"], q["x"])


# ------------------------------------------------------------------ orthogonal rows (1 and 4)
@pytest.mark.parametrize("row1", [False, True])
@pytest.mark.parametrize("m,k", [(5, 3), (9, 1), (6, 5)])
def test_orthogonal_matches_brute_force(rng, row1, m, k):
    """Table 1 rows 4 / 1 (Krylov operator (I - WW^T) A) with the per-cycle Galerkin
    completion (R19): per-step equality with lstsq over the explicit space."""
    n = 36
    D = random_nonsym(n, rng, shift=1.6)
    W = _orthonormal(n, k, rng)
    b = rng.standard_normal(n)
    var = "orthogonal_aug" if row1 else "orthogonal"
    r = oracle.solve(oracle.Matrix.from_dense(D), b, m=m, variant=var, W=W, tol=1e-9, max_iters=800)
    xb, itb, hb = restarted_oblique(D, b, m, W, tol=1e-9, max_iters=800, row2=row1, orth=True)
    assert r["converged"]
    assert r["iterations"] == itb
    kk = min(len(hb), len(r["history"]))
    assert np.allclose(r["history"][:kk], hb[:kk], rtol=1e-7, atol=1e-12)
    assert np.linalg.norm(r["x"] - xb) <= 1e-7 * np.linalg.norm(xb)


def test_orthogonal_rows_1_and_4_coincide_and_converge(rng):
    n, k = 80, 5
    D = random_nonsym(n, rng, shift=1.3)
    W = _orthonormal(n, k, rng)
    b = rng.standard_normal(n)
    A = oracle.Matrix.from_dense(D)
    p = oracle.solve(A, b, m=6, variant="orthogonal", W=W, tol=1e-10, max_iters=3000)
    q = oracle.solve(A, b, m=6, variant="orthogonal_aug", W=W, tol=1e-10, max_iters=3000)
    assert p["converged"] and q["converged"] and p["iterations"] == q["iterations"]
    assert np.linalg.norm(p["x"] - q["x"]) <= 1e-9 * np.linalg.norm(p["x"])
    xs = np.linalg.solve(D, b)
    assert np.linalg.norm(p["x"] - xs) <= 1e-8 * np.linalg.norm(xs)
    assert np.linalg.norm(W.T @ (b - D @ p["x"])) <= 1e-13 * np.linalg.norm(b)


def test_orthogonal_rhs_in_image_of_recycle_space(rng):
    n, k = 30, 4
    D = random_nonsym(n, rng)
    W = _orthonormal(n, k, rng)
    c = rng.standard_normal(k)
    r = oracle.solve(oracle.Matrix.from_dense(D), D @ W @ c, m=10, variant="orthogonal", W=W)
    assert r["iterations"] == 0 and r["converged"]
    assert np.linalg.norm(r["x"] - W @ c) <= 1e-12 * np.linalg.norm(c)
