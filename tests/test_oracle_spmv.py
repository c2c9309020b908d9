"""Pins for the oracle's SpMV (oracle.c or_spmv / or_spmv_row)."""
import numpy as np
import pytest

import oracle


def _dense_from_csr(n, rp, ci, v):
    D = np.zeros((n, n))
    for i in range(n):
        for p in range(rp[i], rp[i + 1]):
            D[i, ci[p]] += v[p]
    return D


def test_identity_closed_form():
    A = oracle.Matrix.from_dense(np.eye(3))
    assert np.array_equal(oracle.spmv(A, [1.0, 2.0, 3.0]), [1.0, 2.0, 3.0])


def test_diagonal_closed_form():
    A = oracle.Matrix.from_dense(np.diag([2.0, 3.0]))
    assert np.array_equal(oracle.spmv(A, [1.0, 1.0]), [2.0, 3.0])


def test_single_entry_shift():
    A = oracle.Matrix(2, [0, 1, 1], [1], [1.0])          # [[0,1],[0,0]]
    assert np.array_equal(oracle.spmv(A, [5.0, 7.0]), [7.0, 0.0])


def test_empty_rows_and_empty_matrix():
    A = oracle.Matrix(4, [0, 0, 2, 2, 3], [0, 3, 1], [1.0, 2.0, 3.0])
    x = np.array([1.0, 10.0, 100.0, 1000.0])
    assert np.array_equal(oracle.spmv(A, x), [0.0, 2001.0, 0.0, 30.0])
    Z = oracle.Matrix(3, [0, 0, 0, 0], np.zeros(0, np.int32), np.zeros(0))
    assert np.array_equal(oracle.spmv(Z, np.ones(3)), np.zeros(3))


@pytest.mark.parametrize("n", [8, 37])
def test_random_vs_dense_brute_force(rng, n):
    D = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.5)
    A = oracle.Matrix.from_dense(D)
    x = rng.standard_normal(n)
    y_bf = np.array([sum(D[i, j] * x[j] for j in range(n)) for i in range(n)])
    assert np.allclose(oracle.spmv(A, x), y_bf, rtol=1e-14, atol=1e-14)
    for i in (0, n // 2, n - 1):
        assert oracle.spmv_row(A, i, x) == oracle.spmv(A, x)[i]


def test_bsr_vs_dense_expansion(rng):
    nb, B = 5, 4
    rp = [0]
    ci = []
    for I in range(nb):
        cols = sorted(set([I] + list(rng.choice(nb, 2, replace=False))))
        ci += cols
        rp.append(len(ci))
    vals = rng.standard_normal(len(ci) * B * B)
    A = oracle.Matrix(nb * B, rp, ci, vals, fmt="bsr", block=B)
    D = np.zeros((nb * B, nb * B))
    for I in range(nb):
        for p in range(rp[I], rp[I + 1]):
            blk = vals[p * B * B:(p + 1) * B * B].reshape(B, B).T   # stored column-major
            D[I * B:(I + 1) * B, ci[p] * B:(ci[p] + 1) * B] += blk
    x = rng.standard_normal(nb * B)
    assert np.allclose(oracle.spmv(A, x), D @ x, rtol=1e-14, atol=1e-13)
    assert oracle.spmv_row(A, 7, x) == oracle.spmv(A, x)[7]
