"""Pins for the oracle's plain restarted GMRES(m) (oracle.c or_solve, variant plain;
PAPER.md:133-135 minimal residual, 171-175 GMRES, 36-38 restart)."""
import numpy as np
import pytest

import oracle
from bruteforce import random_nonsym, restarted_minres


def test_identity_one_iteration(rng):
    b = rng.standard_normal(10)
    r = oracle.solve(oracle.Matrix.from_dense(np.eye(10)), b, m=5)
    assert r["iterations"] == 1 and r["converged"]
    assert np.allclose(r["x"], b, rtol=0, atol=1e-15)


def test_scaled_identity(rng):
    b = rng.standard_normal(10)
    r = oracle.solve(oracle.Matrix.from_dense(2 * np.eye(10)), b, m=5)
    assert r["iterations"] == 1
    assert np.allclose(r["x"], b / 2, rtol=0, atol=1e-15)


@pytest.mark.parametrize("n", [20, 30])
def test_dense_lu_oracle(rng, n):
    D = np.diag(n + rng.random(n)) + rng.standard_normal((n, n))
    b = rng.standard_normal(n)
    r = oracle.solve(oracle.Matrix.from_dense(D), b, m=n, tol=1e-12)
    xs = np.linalg.solve(D, b)
    assert r["converged"]
    assert np.linalg.norm(r["x"] - xs) <= 1e-10 * np.linalg.norm(xs)


def test_restart_n_terminates_within_n(rng):
    n = 25
    D = random_nonsym(n, rng, shift=1.2)
    b = rng.standard_normal(n)
    r = oracle.solve(oracle.Matrix.from_dense(D), b, m=n, tol=1e-6)
    assert r["converged"] and r["iterations"] <= n and r["cycles"] == 1


def test_converged_initial_guess_zero_iterations(rng):
    n = 15
    D = random_nonsym(n, rng)
    xs = rng.standard_normal(n)
    r = oracle.solve(oracle.Matrix.from_dense(D), D @ xs, x0=xs, m=5)
    assert r["iterations"] == 0 and r["converged"]


def test_zero_rhs():
    r = oracle.solve(oracle.Matrix.from_dense(np.eye(4) * 3), np.zeros(4), x0=np.ones(4))
    assert r["converged"] and r["iterations"] == 0 and np.all(r["x"] == 0)


@pytest.mark.parametrize("m", [1, 4, 7])
def test_matches_brute_force_restarted_minres(rng, m):
    """Every step's residual equals the explicit least-squares minimum over x_c + K_j(A, r_c)
    (numpy lstsq over an explicit Krylov basis) — pins the definition, restarts included."""
    n = 30
    D = random_nonsym(n, rng, shift=1.6)
    b = rng.standard_normal(n)
    r = oracle.solve(oracle.Matrix.from_dense(D), b, m=m, tol=1e-9, max_iters=400)
    xb, itb, hb = restarted_minres(D, b, m, tol=1e-9, max_iters=400)
    assert r["iterations"] == itb
    k = min(len(hb), len(r["history"]))
    assert np.allclose(r["history"][:k], hb[:k], rtol=1e-7, atol=1e-12)
    assert np.linalg.norm(r["x"] - xb) <= 1e-7 * np.linalg.norm(xb)


def test_history_nonincreasing_within_cycle(rng):
    n = 40
    D = random_nonsym(n, rng, shift=1.3)
    b = rng.standard_normal(n)
    m = 8
    r = oracle.solve(oracle.Matrix.from_dense(D), b, m=m, tol=1e-10, max_iters=300)
    h = r["history"]
    for c0 in range(0, len(h), m):
        seg = h[c0:c0 + m]
        assert np.all(np.diff(seg) <= 1e-14), seg
    # and the true residual never increases across cycles (each cycle's space contains 0)
    ends = h[m - 1::m]
    assert np.all(np.diff(ends) <= 1e-14)


def test_final_true_residual_meets_tol(rng):
    n = 50
    D = random_nonsym(n, rng, shift=1.5)
    b = rng.standard_normal(n)
    r = oracle.solve(oracle.Matrix.from_dense(D), b, m=10, tol=1e-8)
    assert r["converged"]
    assert np.linalg.norm(b - D @ r["x"]) / np.linalg.norm(b) <= 1e-8
