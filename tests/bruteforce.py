"""Brute-force numpy references used to PIN the oracle on tiny inputs.

Independent of ``oracle/`` (no shared code): dense matrices, explicit spaces, LAPACK least squares
(``numpy.linalg.lstsq``), Householder QR (``numpy.linalg.qr``) and the literal projector formula of
PAPER.md Table 1 row 6 (``I - AV(V^T A^T A V)^{-1} V^T A^T``).  Small n only.
"""
import numpy as np


def ls_projector(A, W):
    """P = I - AW((AW)^T AW)^{-1}(AW)^T, written literally."""
    C = A @ W
    return np.eye(A.shape[0]) - C @ np.linalg.inv(C.T @ C) @ C.T


def _orth_append(K, v):
    """Return an orthonormal basis of span(K, v) (Householder QR of the stacked matrix)."""
    M = np.column_stack(K + [v])
    Q, _ = np.linalg.qr(M)
    return [Q[:, i] for i in range(Q.shape[1])]


def ssor_matrix(A, order, omega):
    """The SSOR preconditioner matrix, assembled literally: in the row order `order`,
    M_p = (D + wL) D^{-1} (D + wU) / (w (2 - w)) with A_p = A[order][:, order] = D + L + U;
    returned in the original indexing (M[order][:, order] = M_p)."""
    order = np.asarray(order)
    Ap = A[np.ix_(order, order)]
    D = np.diag(np.diag(Ap))
    L = np.tril(Ap, -1)
    U = np.triu(Ap, 1)
    Mp = (D + omega * L) @ np.linalg.inv(D) @ (D + omega * U) / (omega * (2.0 - omega))
    M = np.empty_like(Mp)
    M[np.ix_(order, order)] = Mp
    return M


def restarted_minres(A, b, m, variant="plain", W=None, tol=1e-8, max_iters=2000, x0=None, Minv=None):
    """x_{c,j} = argmin over x_c (+ span W) + Minv K_j(op, v) of ||b - A x||, cycle by cycle.

    op/v: plain, augment -> (A Minv, r_c); deflate -> (P A Minv, P r_c) (Minv = I without a
    preconditioner).  Start for recycled variants: x_0 <- x0 + W lstsq(AW, r(x0)).
    Returns (x, iterations, history)."""
    Mi = np.eye(A.shape[0]) if Minv is None else Minv
    n = A.shape[0]
    bn = np.linalg.norm(b)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=float)
    rec = variant != "plain" and W is not None and W.shape[1] > 0
    if rec:
        C = A @ W
        x = x + W @ np.linalg.lstsq(C, b - A @ x, rcond=None)[0]
        P = ls_projector(A, W)
    hist, iters = [], 0
    while True:
        r = b - A @ x
        if np.linalg.norm(r) / bn <= tol or iters >= max_iters:
            break
        if variant == "deflate" and rec:
            op, v = P @ A @ Mi, P @ r
        else:
            op, v = A @ Mi, r
        K = [v / np.linalg.norm(v)]
        for j in range(m):
            S = np.column_stack(([W[:, i] for i in range(W.shape[1])] if rec else []) + [Mi @ q for q in K])
            y = np.linalg.lstsq(A @ S, r, rcond=None)[0]
            res = np.linalg.norm(r - A @ S @ y)
            hist.append(res / bn)
            iters += 1
            if res / bn <= tol or j == m - 1 or iters >= max_iters:
                x = x + S @ y
                break
            K = _orth_append(K, op @ K[-1])
    return x, iters, np.array(hist)


def oblique_projector(A, W):
    """M_D = I - A W E^{-1} W^T with E = W^T A W, written literally (Table 1 rows 2/5)."""
    return np.eye(A.shape[0]) - A @ W @ np.linalg.inv(W.T @ A @ W) @ W.T


def restarted_oblique(A, b, m, W, tol=1e-8, max_iters=2000, row2=False, Minv=None, orth=False):
    """Table 1 rows 5 (row2=False) / 2 (row2=True) with the Galerkin start at every cycle
    (R15): x_c <- x_c + W E^{-1} W^T r(x_c); z = argmin over K_j(M_D A, v) of
    ||M_D r_c - M_D A z|| with v = M_D r_c (row 5) or r_c (row 2).  Returns (x, iterations, history)."""
    n = A.shape[0]
    bn = np.linalg.norm(b)
    x = np.zeros(n)
    E = W.T @ A @ W
    # Krylov projector: oblique M_D (rows 2/5) or the literal orthogonal I - W W^T (rows 1/4)
    M = np.eye(A.shape[0]) - W @ W.T if orth else oblique_projector(A, W)
    Mi = np.eye(A.shape[0]) if Minv is None else Minv
    MA = M @ A @ Mi
    hist, iters = [], 0
    while True:
        x = x + W @ np.linalg.solve(E, W.T @ (b - A @ x))
        r = b - A @ x
        if np.linalg.norm(r) / bn <= tol or iters >= max_iters:
            break
        rh = M @ r
        v = r if row2 else rh
        K = [v / np.linalg.norm(v)]
        for j in range(m):
            S = np.column_stack(K)
            y = np.linalg.lstsq(MA @ S, rh, rcond=None)[0]
            res = np.linalg.norm(rh - MA @ S @ y)
            hist.append(res / bn)
            iters += 1
            if res / bn <= tol or j == m - 1 or iters >= max_iters:
                x = x + Mi @ (S @ y)
                break
            K = _orth_append(K, MA @ K[-1])
    return x, iters, np.array(hist)


def random_nonsym(n, rng, shift=2.5, density=1.0):
    """Dense non-symmetric test matrix shift*I + G/sqrt(n) (eigenvalues in a disc around shift)."""
    G = rng.standard_normal((n, n)) / np.sqrt(n)
    if density < 1.0:
        G *= rng.random((n, n)) < density
    return shift * np.eye(n) + G
