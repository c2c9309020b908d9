"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star):
  pattern / indices        bit-exact
  SpMV                     ||y_g - y_o|| <= 1e-13 ||y_o||  and componentwise <= 1e-13 (|A||x|)
  singular values          |d sigma_i| <= max(1e-10 sigma_i, 1e-15 sigma_1)
  solutions at tol 1e-8    ||x_g - x_o|| <= 1e-7 ||x_o||
  iteration counts         within +-2
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def make_ctx(hm, cfg=None, sell=False, max_m=64, s=16, k=8, flags=0):
    from paper_1807_09467_b200 import Context
    return Context(hm.n, t(hm.row_ptr), t(hm.col_idx), t(hm.val), fmt=hm.fmt, block=hm.block,
                   sell_C=32 if sell else 0, max_m=max_m, max_snapshots=s, max_k=k, flags=flags)


def random_csr(n, rng, per_row=(0, 9), diag=4.0):
    rp = [0]
    ci, v = [], []
    for i in range(n):
        nr = rng.integers(per_row[0], per_row[1] + 1)
        cols = set(rng.choice(n, size=min(nr, n), replace=False).tolist()) | {i}
        for c in sorted(cols):
            ci.append(c)
            v.append(diag if c == i else rng.standard_normal() / np.sqrt(max(nr, 1)))
        rp.append(len(ci))
    return synth.HostMatrix("csr", n, np.array(rp, np.int32), np.array(ci, np.int32), np.array(v))


def spmv_check(hm, x, y):
    yo = oracle.spmv(oracle.Matrix.from_host(hm), x)
    S = hm.to_scipy()
    ax = abs(S) @ np.abs(x)
    assert np.linalg.norm(y - yo) <= 1e-13 * np.linalg.norm(yo)
    assert np.all(np.abs(y - yo) <= 1e-13 * ax + 1e-300)


# ------------------------------------------------------------------------------------- SpMV
@pytest.mark.parametrize("n", [1, 31, 1000, 4097])
@pytest.mark.parametrize("sell", [False, True])
def test_spmv_random_ragged(n, sell, rng):
    hm = random_csr(n, rng, per_row=(0, 40) if n > 100 else (0, 5))
    ctx = make_ctx(hm, sell=sell)
    x = rng.standard_normal(n)
    y = torch.zeros(n, dtype=torch.float64, device=DEV)
    ctx.apply(t(x), y)
    spmv_check(hm, x, y.cpu().numpy())
    yh = np.zeros(n)
    ctx.apply(x, yh)                   # host-pointer path
    assert np.array_equal(yh, y.cpu().numpy())


@pytest.mark.parametrize("name,N", [("C1", 32), ("C2", 512), ("C3", 256), ("C4", 40), ("C5", 3)])
def test_spmv_configs(name, N, rng):
    cfg = synth.CONFIGS[name].reduced(N)
    seq = synth.HostSequence(cfg)
    hm = seq.matrix(2, seq.initial())
    ctx = make_ctx(hm, sell=cfg.fmt == "sell")
    x = rng.standard_normal(cfg.n)
    y = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
    ctx.apply(t(x), y)
    spmv_check(hm, x, y.cpu().numpy())


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_spmv_full_size_sampled_rows(name, rng):
    """Full BASELINE size, in the launch configuration the bench uses: sampled rows against the
    oracle's single-row product."""
    cfg = synth.CONFIGS[name]
    seq = synth.HostSequence(cfg)
    hm = seq.matrix(1, seq.initial())
    ctx = make_ctx(hm, sell=cfg.fmt == "sell")
    x = rng.standard_normal(cfg.n)
    y = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
    ctx.apply(t(x), y)
    y = y.cpu().numpy()
    M = oracle.Matrix.from_host(hm)
    rows = np.concatenate([[0, 1, cfg.n - 1], rng.integers(0, cfg.n, 2000)])
    for r in rows:
        yo = oracle.spmv_row(M, int(r), x)
        assert abs(y[r] - yo) <= 1e-13 * (np.abs(hm.val[hm.row_ptr[r]:hm.row_ptr[r + 1]]) @
                                         np.abs(x[hm.col_idx[hm.row_ptr[r]:hm.row_ptr[r + 1]]]))


# ------------------------------------------------------------------------------------- solves
@pytest.mark.parametrize("variant", ["plain", "augment", "deflate", "oblique", "orthogonal"])
@pytest.mark.parametrize("n,m,k", [(200, 10, 4), (1023, 25, 8), (64, 64, 3)])
def test_solve_random_vs_oracle(variant, n, m, k, rng):
    hm = random_csr(n, rng, per_row=(2, 8), diag=2.2)
    W = np.linalg.qr(rng.standard_normal((n, k)))[0]
    b = rng.standard_normal(n)
    ctx = make_ctx(hm, max_m=max(m, 8), s=k, k=k)
    for i in range(k):
        ctx.push_snapshot(t(W[:, i] * (k - i)))
    ke, sig = ctx.build_recycle(k)
    assert ke == k
    Wg = np.zeros((k, n))
    ctx.export(0, Wg)
    Wg = Wg.T
    x = torch.zeros(n, dtype=torch.float64, device=DEV)
    rep = ctx.solve(t(b), x, m=m, variant=variant, tol=1e-8, history_cap=5000)
    ref = oracle.solve(oracle.Matrix.from_host(hm), b, m=m, variant=variant, W=W, tol=1e-8)
    xg = x.cpu().numpy()
    assert rep["converged"] and ref["converged"]
    assert np.linalg.norm(xg - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])
    assert abs(rep["iterations"] - ref["iterations"]) <= 2
    # true residual from the oracle's SpMV
    r = b - oracle.spmv(oracle.Matrix.from_host(hm), xg)
    assert np.linalg.norm(r) / np.linalg.norm(b) <= 1e-8
    assert abs(rep["rel_residual"] - np.linalg.norm(r) / np.linalg.norm(b)) <= 1e-12
    # span(W_gpu) == span(W)
    assert np.linalg.norm(Wg @ Wg.T - W @ W.T, 2) <= 1e-10
    h = rep["history"]
    assert len(h) == rep["iterations"]
    if variant in ("oblique", "orthogonal"):  # final Galerkin correction: W^T (b - A x) = 0
        assert np.linalg.norm(W.T @ r) <= 1e-11 * np.linalg.norm(b)
        kk = min(len(h), len(ref["history"]))   # Givens estimates vs the oracle's explicit minima
        assert np.allclose(h[:kk], ref["history"][:kk], rtol=1e-5, atol=1e-11)


def test_b_zero_and_converged_x0(rng):
    hm = random_csr(100, rng)
    ctx = make_ctx(hm)
    x = torch.ones(100, dtype=torch.float64, device=DEV)
    rep = ctx.solve(torch.zeros(100, dtype=torch.float64, device=DEV), x, x0=x.clone(), m=10)
    assert rep["converged"] and rep["iterations"] == 0 and float(x.abs().max()) == 0.0
    xs = rng.standard_normal(100)
    b = hm.to_scipy() @ xs
    x2 = torch.zeros(100, dtype=torch.float64, device=DEV)
    rep = ctx.solve(t(b), x2, x0=t(xs), m=10)
    assert rep["converged"] and rep["iterations"] == 0


@pytest.mark.parametrize("n", [1024, 1000])   # n = n_pad (caller buffers used in place) / padded
def test_initial_guess_and_buffer_modes_agree(n, rng):
    """The persistent solve reads b and iterates x in the caller's device buffers when n = n_pad;
    every way of passing x0 (none, a separate device buffer, in place in x_out, host buffers) gives
    the same iterates, and the result is the oracle's."""
    hm = random_csr(n, rng, per_row=(2, 6))
    ctx = make_ctx(hm)
    b = rng.standard_normal(n)
    x0 = 0.1 * rng.standard_normal(n)
    ref = oracle.solve(oracle.Matrix.from_host(hm), b, m=20, x0=x0, tol=1e-8)
    outs = []
    xa = torch.zeros(n, dtype=torch.float64, device=DEV)              # separate x0 buffer
    outs.append((ctx.solve(t(b), xa, x0=t(x0), m=20), xa.cpu().numpy()))
    xb = t(x0)                                                        # in place: x0 is x_out
    outs.append((ctx.solve(t(b), xb, x0=xb, m=20), xb.cpu().numpy()))
    xc = np.zeros(n)                                                  # host buffers
    outs.append((ctx.solve(b, xc, x0=x0, m=20), xc))
    for rep, x in outs:
        assert rep["converged"]
        assert rep["iterations"] == outs[0][0]["iterations"]
        assert np.array_equal(x, outs[0][1])                          # bitwise: same kernels, same inputs
        assert np.linalg.norm(x - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])
        assert abs(rep["iterations"] - ref["iterations"]) <= 2
    xd = torch.full((n,), 7.0, dtype=torch.float64, device=DEV)       # x0 = None: zero start, x_out overwritten
    rep = ctx.solve(t(b), xd, m=20)
    ref0 = oracle.solve(oracle.Matrix.from_host(hm), b, m=20, tol=1e-8)
    assert rep["converged"] and abs(rep["iterations"] - ref0["iterations"]) <= 2
    assert np.linalg.norm(xd.cpu().numpy() - ref0["x"]) <= 1e-7 * np.linalg.norm(ref0["x"])


def test_persistent_refusal_falls_back_with_caller_buffers(rng):
    """n = n_pad with device buffers but m > 64: the persistent kernel refuses the launch after the
    caller's b / x were chosen as its buffers; the graph path then gets the library's copies."""
    n, m = 4096, 100
    hm = random_csr(n, rng, per_row=(2, 6), diag=2.0)
    ctx = make_ctx(hm, max_m=m)
    b = rng.standard_normal(n)
    x0 = 0.1 * rng.standard_normal(n)
    x = t(x0)                                                         # in place
    rep = ctx.solve(t(b), x, x0=x, m=m, tol=1e-9)
    ref = oracle.solve(oracle.Matrix.from_host(hm), b, m=m, x0=x0, tol=1e-9)
    assert rep["converged"] and abs(rep["iterations"] - ref["iterations"]) <= 2
    assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])


def test_max_iters_cap_reports_not_converged(rng):
    hm = random_csr(500, rng, diag=1.0)
    ctx = make_ctx(hm)
    x = torch.zeros(500, dtype=torch.float64, device=DEV)
    rep = ctx.solve(t(rng.standard_normal(500)), x, m=5, tol=1e-14, max_iters=7)
    assert rep["iterations"] == 7 and not rep["converged"]


def test_rhs_in_image_of_recycle_space(rng):
    n, k = 300, 4
    hm = random_csr(n, rng)
    W = np.linalg.qr(rng.standard_normal((n, k)))[0]
    ctx = make_ctx(hm, s=k, k=k)
    for i in range(k):
        ctx.push_snapshot(t(W[:, i] * (i + 1)))
    ctx.build_recycle(k)
    c = rng.standard_normal(k)
    b = hm.to_scipy() @ (W @ c)
    for v in ("augment", "deflate", "oblique", "orthogonal"):
        x = torch.zeros(n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b), x, m=10, variant=v)
        assert rep["iterations"] == 0 and rep["converged"]
        assert np.linalg.norm(x.cpu().numpy() - W @ c) <= 1e-10 * np.linalg.norm(c)


def test_bitwise_deterministic(rng):
    cfg = synth.CONFIGS["C2"].reduced(128)
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    hm = seq.matrix(1, u)
    b = seq.rhs(1, u)
    outs = []
    for _ in range(2):
        ctx = make_ctx(hm, max_m=cfg.m)
        x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
        ctx.solve(t(b), x, m=cfg.m)
        outs.append(x.cpu().numpy())
        ctx.close()
    assert np.array_equal(outs[0], outs[1])


# ------------------------------------------------------------------------------------- SVD
def test_singular_values_vs_oracle(rng):
    n, s = 5000, 12
    P = np.linalg.qr(rng.standard_normal((n, s)))[0]
    Q = np.linalg.qr(rng.standard_normal((s, s)))[0]
    true = np.logspace(0, -6, s)
    X = P @ np.diag(true) @ Q.T
    hm = random_csr(n, rng)
    ctx = make_ctx(hm, s=s, k=s)
    for i in range(s):
        ctx.push_snapshot(t(X[:, i]))
    ke, sig = ctx.build_recycle(5)
    _, so, rank, _ = oracle.svd(X)
    sg = sig[:s]
    assert ke == 5
    assert np.all(np.abs(sg - so) <= np.maximum(1e-10 * so, 1e-15 * so[0]))


def test_rank_deficient_window(rng):
    n = 777
    hm = random_csr(n, rng)
    ctx = make_ctx(hm, s=6, k=6)
    a, b2 = rng.standard_normal(n), rng.standard_normal(n)
    for v in (a, b2, a + b2, 2 * a):
        ctx.push_snapshot(t(v))
    ke, sig = ctx.build_recycle(4)
    assert ke == 2


@pytest.mark.parametrize("name,N,sell", [("C4", 14, False), ("C3", 40, True), ("C5", 3, False)])
def test_recycle_operator_thin_qr(name, N, sell, rng):
    """a4: C = A W (single-read SpMM) and its CholQR2 factors: A W = Q R_C, Q^T Q = I,
    checked with the oracle's SpMV on the exported W."""
    cfg = synth.CONFIGS[name].reduced(N)
    seq = synth.HostSequence(cfg)
    hm = seq.matrix(1, seq.initial())
    k = 12
    ctx = make_ctx(hm, sell=sell, s=k, k=k, max_m=cfg.m)
    for i in range(k):
        ctx.push_snapshot(t(rng.standard_normal(cfg.n)))
    ke, _ = ctx.build_recycle(k)
    x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
    ctx.solve(t(rng.standard_normal(cfg.n)), x, m=cfg.m, variant="deflate", max_iters=3)
    W = np.zeros((ke, cfg.n)); ctx.export(0, W); W = W.T
    Q = np.zeros((ke, cfg.n)); ctx.export(1, Q); Q = Q.T
    R = np.zeros((ke, ke)); ctx.export(2, R); R = R.T      # exported column-major
    M = oracle.Matrix.from_host(hm)
    AW = np.column_stack([oracle.spmv(M, W[:, i]) for i in range(ke)])
    assert np.linalg.norm(AW - Q @ R) <= 1e-12 * np.linalg.norm(AW)
    assert np.linalg.norm(Q.T @ Q - np.eye(ke)) <= 1e-12
    assert np.allclose(np.tril(R, -1), 0.0)


@pytest.mark.parametrize("flags", [0, 8, 4])   # persistent, graph (RG_FLAG_NO_PERSIST), classical CGS2
@pytest.mark.parametrize("n,k", [(7, 5), (7, 1), (12, 4), (40, 8)])
def test_augment_search_space_exhaustion(n, k, flags, rng):
    """Augment with k + m > n: at Krylov step j = n - k the space span(W) + K_j is all of R^n, the Cholesky
    factor T of I - G^T G gets a zero diagonal (tau = 0) and that step COMPLETES the solve.  The GPU must
    accept the column (zero projected residual) as the explicit-space oracle does — found by the soak runs of
    the fuzz (tools/soak.sh): ending the cycle at the previous step took 23 iterations where the oracle
    takes 2 (R5)."""
    hm = random_csr(n, rng, per_row=(1, 5), diag=2.5)
    ctx = make_ctx(hm, s=k, k=k, max_m=64, flags=flags)
    W = np.linalg.qr(rng.standard_normal((n, k)))[0]
    for i in range(k):
        ctx.push_snapshot(t(W[:, i] * (k - i)))
    assert ctx.build_recycle(k)[0] == k
    b = rng.standard_normal(n)
    x = torch.zeros(n, dtype=torch.float64, device=DEV)
    rep = ctx.solve(t(b), x, m=min(2 * n, 64), variant="augment", tol=1e-9, max_iters=500)
    ref = oracle.solve(oracle.Matrix.from_host(hm), b, m=min(2 * n, 64), variant="augment", W=W, tol=1e-9, max_iters=500)
    assert rep["converged"] and ref["converged"]
    assert ref["iterations"] <= n - k and rep["restarts"] == 0
    assert abs(rep["iterations"] - ref["iterations"]) <= 1, (rep["iterations"], ref["iterations"])
    assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
    ctx.close()


@pytest.mark.parametrize("k", [1, 7, 8, 9, 16, 17, 24, 25, 33, 34, 35, 41, 49, 57, 64])
def test_bsr_spmm_every_column_group_count(k, rng):
    """a4 on BSR-64: C = A W through the TMA + DMMA SpMM for every number of 8-column groups (1..8) and every
    panel-stride instantiation (widths <= 18, <= 34, <= 66), incl. widths that are not multiples of 8; the
    consumer loop is instantiated per group count and keeps its accumulator chains over a block row.
    A W = Q R_C against the oracle's SpMV on the exported W."""
    cfg = synth.CONFIGS["C5"].reduced(3)
    seq = synth.HostSequence(cfg)
    hm = seq.matrix(1, seq.initial())
    ctx = make_ctx(hm, s=max(k, 1), k=k, max_m=cfg.m)
    for i in range(k):
        ctx.push_snapshot(t(rng.standard_normal(cfg.n)))
    ke, _ = ctx.build_recycle(k)
    assert ke == k
    x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
    ctx.solve(t(rng.standard_normal(cfg.n)), x, m=cfg.m, variant="deflate", max_iters=2)
    W = np.zeros((ke, cfg.n)); ctx.export(0, W); W = W.T
    Q = np.zeros((ke, cfg.n)); ctx.export(1, Q); Q = Q.T
    R = np.zeros((ke, ke)); ctx.export(2, R); R = R.T      # exported column-major
    M = oracle.Matrix.from_host(hm)
    AW = np.column_stack([oracle.spmv(M, W[:, i]) for i in range(ke)])
    assert np.linalg.norm(AW - Q @ R) <= 1e-12 * np.linalg.norm(AW)
    assert np.linalg.norm(Q.T @ Q - np.eye(ke)) <= 1e-11
    ctx.close()


@pytest.mark.parametrize("variant", ["plain", "augment", "deflate", "oblique", "orthogonal"])
def test_persistent_and_graph_paths_agree(variant, rng):
    """The single cooperative-kernel solve and the CUDA-graph solve compute the same iterates
    (same DCGS2 arithmetic, different reduction trees): same iteration counts, x within 1e-10."""
    from paper_1807_09467_b200 import rg as rgb
    cfg = synth.CONFIGS["C2"].reduced(160)
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    hm = seq.matrix(1, u)
    b = seq.rhs(1, u)
    snaps = [rng.standard_normal(cfg.n) for _ in range(4)]
    out = []
    for flags in (0, rgb.RG_FLAG_NO_PERSIST):
        ctx = make_ctx(hm, max_m=cfg.m, s=8, k=4, flags=flags)
        for v in snaps:
            ctx.push_snapshot(t(v))
        ctx.build_recycle(4)
        x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b), x, m=cfg.m, variant=variant, history_cap=1000)
        out.append((rep, x.cpu().numpy()))
        ctx.close()
    (r0, x0), (r1, x1) = out
    assert r0["converged"] and r1["converged"]
    assert r0["iterations"] == r1["iterations"]
    assert np.linalg.norm(x0 - x1) <= 1e-10 * np.linalg.norm(x1)
    assert np.allclose(r0["history"], r1["history"], rtol=1e-8, atol=1e-14)


def test_bsr_generic_block_size(rng):
    """BSR with 16x16 blocks (generic kernel, not the TMA 64x64 path): SpMV and a solve."""
    nb, B = 40, 16
    rp, ci = [0], []
    for I in range(nb):
        cols = sorted(set([I, (I + 1) % nb, (I + 7) % nb]))
        ci += cols
        rp.append(len(ci))
    vals = rng.standard_normal(len(ci) * B * B) * 0.1
    for p in range(len(ci)):
        I = next(i for i in range(nb) if rp[i] <= p < rp[i + 1])
        if ci[p] == I:
            blk = vals[p * B * B:(p + 1) * B * B]
            blk[::B + 1] += 3.0                      # diagonal of a column-major block
    hm = synth.HostMatrix("bsr", nb * B, np.array(rp, np.int32), np.array(ci, np.int32), vals, B)
    ctx = make_ctx(hm)
    x = rng.standard_normal(nb * B)
    y = torch.zeros(nb * B, dtype=torch.float64, device=DEV)
    ctx.apply(t(x), y)
    spmv_check(hm, x, y.cpu().numpy())
    b = rng.standard_normal(nb * B)
    xs = torch.zeros(nb * B, dtype=torch.float64, device=DEV)
    rep = ctx.solve(t(b), xs, m=20)
    ref = oracle.solve(oracle.Matrix.from_host(hm), b, m=20)
    assert rep["converged"] and abs(rep["iterations"] - ref["iterations"]) <= 2
    assert np.linalg.norm(xs.cpu().numpy() - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])


def test_update_matrix_new_pattern_and_validation(rng):
    """rg_update_matrix with a different pattern (re-validated, re-allocated, graphs rebuilt) and
    rejection of invalid patterns from host and device memory with no side effects."""
    from paper_1807_09467_b200 import rg as rgb
    h1 = random_csr(300, rng, per_row=(1, 4))
    h2 = random_csr(300, rng, per_row=(5, 12))
    ctx = make_ctx(h1)
    b = rng.standard_normal(300)
    x = torch.zeros(300, dtype=torch.float64, device=DEV)
    ctx.solve(t(b), x, m=10)
    ctx.update_matrix(t(h2.val), t(h2.row_ptr), t(h2.col_idx))
    rep = ctx.solve(t(b), x, m=10)
    ref = oracle.solve(oracle.Matrix.from_host(h2), b, m=10)
    assert abs(rep["iterations"] - ref["iterations"]) <= 2
    assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])
    bad = h2.col_idx.copy()
    bad[5], bad[6] = bad[6], bad[5]                  # unsorted row
    for mem in ("host", "device"):
        arr = (lambda a: a) if mem == "host" else t
        with pytest.raises(rgb.RgError) as e:
            ctx.update_matrix(arr(h2.val), arr(h2.row_ptr), arr(bad))
        assert e.value.status == rgb.RG_E_INVAL
    y = torch.zeros(300, dtype=torch.float64, device=DEV)   # the context still holds h2
    xx = rng.standard_normal(300)
    ctx.apply(t(xx), y)
    spmv_check(h2, xx, y.cpu().numpy())


@pytest.mark.parametrize("variant", ["deflate", "oblique"])
def test_singular_recycle_operator_reported(variant, rng):
    """A W rank deficient (A annihilates part of span W) -> RG_E_SINGULAR and the recycle space is
    cleared (E_s may be singular)."""
    from paper_1807_09467_b200 import rg as rgb
    n = 200
    D = np.ones(n) * 2.0
    D[:50] = 0.0                                     # A e_i = 0 for i < 50
    hm = synth.HostMatrix("csr", n, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), D)
    ctx = make_ctx(hm, s=4, k=4)
    for i in range(3):
        v = np.zeros(n)
        v[i] = 1.0                                   # snapshots inside the null space of A
        ctx.push_snapshot(t(v))
    ctx.push_snapshot(t(rng.standard_normal(n)))
    ke, _ = ctx.build_recycle(4)
    assert ke == 4
    x = torch.zeros(n, dtype=torch.float64, device=DEV)
    with pytest.raises(rgb.RgError) as e:
        ctx.solve(t(rng.standard_normal(n)), x, m=10, variant=variant)
    assert e.value.status == rgb.RG_E_SINGULAR
    W = np.zeros((4, n))
    with pytest.raises(rgb.RgError) as e:
        ctx.export(0, W)                             # cleared
    assert e.value.status == rgb.RG_E_STATE


@pytest.mark.parametrize("variant", ["augment", "deflate", "oblique", "orthogonal"])
def test_dcgs2_and_cgs2_paths_agree(variant, rng):
    """Delayed CGS2 (one reduction per step; the oblique projection folded into its coefficients)
    and classical CGS2 (explicit M_D A v_j) give the same iterates."""
    from paper_1807_09467_b200 import rg as rgb
    cfg = synth.CONFIGS["C2"].reduced(160)
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    hm = seq.matrix(1, u)
    b = seq.rhs(1, u)
    snaps = [rng.standard_normal(cfg.n) for _ in range(6)]
    out = []
    for flags in (rgb.RG_FLAG_NO_PERSIST, rgb.RG_FLAG_CGS2):
        ctx = make_ctx(hm, max_m=cfg.m, s=8, k=6, flags=flags)
        for v in snaps:
            ctx.push_snapshot(t(v))
        ctx.build_recycle(6)
        x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b), x, m=cfg.m, variant=variant, history_cap=1000)
        out.append((rep, x.cpu().numpy()))
        ctx.close()
    (r0, x0), (r1, x1) = out
    assert r0["converged"] and r1["converged"]
    assert abs(r0["iterations"] - r1["iterations"]) <= 1
    assert np.linalg.norm(x0 - x1) <= 1e-8 * np.linalg.norm(x1)


@pytest.mark.parametrize("variant,k", [("plain", 0), ("augment", 64), ("deflate", 64), ("oblique", 32)])
def test_maximum_restart_and_recycle_dimension(variant, k, rng):
    """max_m = 128 and max_k = 64 (32 for oblique): the largest reductions ([Q|V] dots of 2(k+m)+2
    values) and the largest least-squares state, against the oracle."""
    n, m = 3000, 128
    hm = random_csr(n, rng, per_row=(2, 8), diag=1.3)
    kk = max(k, 1)
    W = np.linalg.qr(rng.standard_normal((n, kk)))[0]
    b = rng.standard_normal(n)
    ctx = make_ctx(hm, max_m=m, s=64, k=64)
    if k:
        for i in range(k):
            ctx.push_snapshot(t(W[:, i] * (k - i)))
        assert ctx.build_recycle(k)[0] == k
    x = torch.zeros(n, dtype=torch.float64, device=DEV)
    rep = ctx.solve(t(b), x, m=m, variant=variant, tol=1e-10, history_cap=5000)
    ref = oracle.solve(oracle.Matrix.from_host(hm), b, m=m, variant=variant, W=W if k else None, tol=1e-10)
    assert rep["converged"] and ref["converged"]
    assert abs(rep["iterations"] - ref["iterations"]) <= 2
    assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-8 * np.linalg.norm(ref["x"])


def test_variant_switching_on_one_context(rng):
    """One context, one recycle space, the variants in turn: the C = A W / Q / E^{-1} state is
    rebuilt whenever the variant family changes (LS projection vs Galerkin start)."""
    n, m, k = 3000, 20, 5
    hm = random_csr(n, rng, per_row=(2, 8), diag=2.0)
    W = np.linalg.qr(rng.standard_normal((n, k)))[0]
    ctx = make_ctx(hm, max_m=m, s=k, k=k)
    for i in range(k):
        ctx.push_snapshot(t(W[:, i] * (k - i)))
    assert ctx.build_recycle(k)[0] == k
    M = oracle.Matrix.from_host(hm)
    for variant in ("deflate", "oblique", "augment", "orthogonal", "deflate", "oblique", "plain"):
        b = rng.standard_normal(n)
        x = torch.zeros(n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b), x, m=m, variant=variant, tol=1e-9)
        ref = oracle.solve(M, b, m=m, variant=variant, W=None if variant == "plain" else W, tol=1e-9)
        assert rep["converged"] and ref["converged"], variant
        assert abs(rep["iterations"] - ref["iterations"]) <= 2, (variant, rep["iterations"], ref["iterations"])
        assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"]), variant


@pytest.mark.parametrize("variant", ["plain", "augment", "deflate", "oblique"])
def test_persistent_multi_cta_wide_pattern(variant, rng):
    """A random pattern couples every row range with every other one, so the persistent solve's
    neighbour synchronisation must wait on all CTAs (n = 20,000: many CTAs)."""
    from paper_1807_09467_b200 import rg as rgb
    n, m, k = 20000, 25, 4
    hm = random_csr(n, rng, per_row=(3, 7), diag=2.4)
    W = np.linalg.qr(rng.standard_normal((n, k)))[0]
    b = rng.standard_normal(n)
    outs = []
    for flags in (0, rgb.RG_FLAG_NO_PERSIST):
        ctx = make_ctx(hm, max_m=m, s=k, k=k, flags=flags)
        for i in range(k):
            ctx.push_snapshot(t(W[:, i] * (k - i)))
        ctx.build_recycle(k)
        x = torch.zeros(n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b), x, m=m, variant=variant, tol=1e-9)
        outs.append((rep, x.cpu().numpy()))
        ctx.close()
    ref = oracle.solve(oracle.Matrix.from_host(hm), b, m=m, variant=variant, W=None if variant == "plain" else W,
                       tol=1e-9)
    for rep, xg in outs:
        assert rep["converged"] and abs(rep["iterations"] - ref["iterations"]) <= 2
        assert np.linalg.norm(xg - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])


# ------------------------------------------------------------------------- asynchronous recycle build
@pytest.mark.parametrize("variant", ["deflate", "augment"])
def test_deferred_build_matches_synchronous(variant, rng):
    """rg_build_recycle with k_eff = sigma = NULL (asynchronous, finished inside the next rg_solve)
    gives bit-identical solves to the synchronous call, also when a snapshot is pushed between the
    build and its solve (the build reads the window in stream order)."""
    cfg = synth.CONFIGS["C1"]
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    A1 = seq.matrix(1, u)
    ctxs = [make_ctx(A1, max_m=cfg.m, s=cfg.s, k=cfg.k) for _ in range(2)]
    xs = [torch.zeros(cfg.n, dtype=torch.float64, device=DEV) for _ in range(2)]
    extra = t(rng.standard_normal(cfg.n))
    for step in range(1, 6):
        A = seq.matrix(step, u)
        b = t(seq.rhs(step, u))
        reps = []
        for i, (ctx, x) in enumerate(zip(ctxs, xs)):
            ctx.update_matrix(t(A.val))
            if step > 1:
                if i == 0:
                    ke, _ = ctx.build_recycle(cfg.k)
                    assert ke >= 1
                else:
                    assert ctx.build_recycle(cfg.k, deferred=True) == (None, None)
                if step == 3:
                    ctx.push_snapshot(extra)
            x.zero_()
            reps.append(ctx.solve(b, x, m=cfg.m, variant=variant, tol=cfg.tol))
        assert reps[0]["iterations"] == reps[1]["iterations"], reps
        assert reps[0]["converged"] and reps[1]["converged"]
        assert torch.equal(xs[0], xs[1])
        u = xs[0].cpu().numpy()
        for ctx in ctxs:
            ctx.push_snapshot(t(u))
    for ctx in ctxs:
        ctx.close()


@pytest.mark.parametrize("flags,exact", [(4 | 8, True), (8, False), (0, False)])   # CGS2 graph / DCGS2 graph / persistent
@pytest.mark.parametrize("variant", ["plain", "deflate"])
def test_spmv_count_is_counted(flags, exact, variant):
    """rg_report.spmv_count is counted by the kernels that run the products (not a formula).  With
    classical CGS2 every Arnoldi step is one SpMV and every cycle start but the first (x0 = 0: r = b)
    one residual SpMV: iterations + restarts + 1, plus k_eff for C = A W; DCGS2 may issue one extra
    product per cycle (the step after the stopping column), the persistent kernel also forms A x0."""
    cfg = synth.CONFIGS["C1"]
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    hm = seq.matrix(1, u)
    ctx = make_ctx(hm, max_m=cfg.m, s=cfg.s, k=cfg.k, flags=flags)
    x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
    for i in range(4):
        ctx.solve(t(seq.rhs(1, u) * (1 + 0.2 * i)), x, m=12, variant="plain", tol=1e-8)
        ctx.push_snapshot(x)
    k = 0
    if variant == "deflate":
        k, _ = ctx.build_recycle(3)
    b = seq.rhs(1, u) * 1.7 + np.random.default_rng(4).standard_normal(cfg.n)   # not in the window's span
    rep = ctx.solve(t(b), x, m=6, variant=variant, tol=1e-8)
    assert rep["converged"] and rep["restarts"] >= 1 and rep["k_eff"] == k
    # cycle starts: restarts + 2, minus the first one's A x0 when x0 = 0 on the graph path (r = b, no product)
    base = rep["iterations"] + rep["restarts"] + 1 + k
    if exact:
        assert rep["spmv_count"] == base, rep
    else:
        assert base <= rep["spmv_count"] <= base + rep["restarts"] + 2, rep
    ctx.close()


def test_orthogonalisation_switch_inside_one_context(rng):
    """The graph path picks DCGS2 or classical CGS2 per solve (one SpMV vs one basis pass,
    8 n (k_eff + m + 2) bytes), and the solve graph is cached per choice (a graph
    captured for one choice must never be replayed for the other).  One context, graph path, a
    deflate sequence whose k_eff grows across the threshold and back down, and m changing between
    solves: every solve against the oracle, and both orthogonalisations observed."""
    from paper_1807_09467_b200 import rg as rgb
    n = 3000
    hm = random_csr(n, rng, per_row=(4, 6), diag=2.5)     # ~6 entries/row
    M = oracle.Matrix.from_host(hm)
    kmax = 8
    basis = np.linalg.qr(rng.standard_normal((n, kmax)))[0]
    ctx = make_ctx(hm, max_m=16, s=kmax, k=kmax, flags=rgb.RG_FLAG_NO_PERSIST | rgb.RG_FLAG_PROFILE)
    seen = set()
    # (k_eff, m): 8 n (k + m + 2) vs ~92 n bytes of A (+ x, y) -> CGS2 below, DCGS2 above
    plan = [(1, 4), (3, 4), (8, 4), (2, 4), (0, 4), (0, 12), (8, 12), (1, 4), (6, 8)]
    for k, m in plan:
        ctx.clear_snapshots()
        for i in range(k):
            ctx.push_snapshot(t(basis[:, i] * (k - i)))
        if k:
            assert ctx.build_recycle(k)[0] == k
        variant = "deflate" if k else "plain"
        b = rng.standard_normal(n)
        ctx.reset_kernel_stats()
        x = torch.zeros(n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b), x, m=m, variant=variant, tol=1e-9)
        ks = ctx.kernel_stats()
        dc = ks["dcgs_dots_ls"]["launches"] > 0
        cg = ks["orth_upd_norm_ls"]["launches"] > 0
        assert dc != cg, (k, m, ks["dcgs_dots_ls"], ks["orth_upd_norm_ls"])
        seen.add("dcgs2" if dc else "cgs2")
        a_bytes = 12 * len(hm.val) + 4 * (n + 1) + 16 * n   # the library's byte model of one SpMV
        assert dc == (a_bytes <= 8 * n * (k + m + 2)), (k, m, dc)
        ref = oracle.solve(M, b, m=m, variant=variant, W=basis[:, :k] if k else None, tol=1e-9)
        assert rep["converged"] and ref["converged"], (k, m)
        assert abs(rep["iterations"] - ref["iterations"]) <= 2, (k, m, rep["iterations"], ref["iterations"])
        assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"]), (k, m)
    assert seen == {"dcgs2", "cgs2"}
    ctx.close()


@pytest.mark.parametrize("variant", ["plain", "augment", "deflate"])
def test_cgs2_tma_passes_vs_oracle(variant, rng):
    """Classical CGS2 on the graph path at a size where its passes run TMA-staged (n_pad >= 148 x 512
    rows: k_cgs_tma for D1 / UD2 / UN and the cycle-start CS_DQ / CS_UN), against the oracle, with
    restarts and the recycle space of a window of earlier solutions."""
    from paper_1807_09467_b200 import rg as rgb
    cfg = synth.CONFIGS["C2"].reduced(320)            # n = 102,400
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    hm = seq.matrix(1, u)
    b = seq.rhs(1, u)
    M = oracle.Matrix.from_host(hm)
    k = 6
    snaps = [oracle.solve(M, seq.rhs(1, u) + 0.1 * i * rng.standard_normal(cfg.n), m=cfg.m, tol=1e-6)["x"]
             for i in range(k)]
    m = 20                                             # restarts inside the solve
    ctx = make_ctx(hm, max_m=m, s=k, k=k, flags=rgb.RG_FLAG_CGS2 | rgb.RG_FLAG_NO_PERSIST)
    W = None
    if variant != "plain":
        for v in snaps:
            ctx.push_snapshot(t(v))
        ke, _ = ctx.build_recycle(k)
        W, _, _ = oracle.recycle_basis(np.stack(snaps, 1), k)
        assert ke == W.shape[1]
    x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
    rep = ctx.solve(t(b), x, m=m, variant=variant, tol=cfg.tol, history_cap=5000)
    ref = oracle.solve(M, b, m=m, variant=variant, W=W, tol=cfg.tol)
    assert rep["converged"] and ref["converged"]
    assert abs(rep["iterations"] - ref["iterations"]) <= 2, (rep["iterations"], ref["iterations"])
    xg = x.cpu().numpy()
    assert np.linalg.norm(xg - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])
    r = b - oracle.spmv(M, xg)
    assert np.linalg.norm(r) / np.linalg.norm(b) <= cfg.tol
    ctx.close()


def test_kernel_trace_timeline(rng):
    """rg_kernel_trace (RG_FLAG_PROFILE): every kernel start has a matching end or is a no-op, times are
    ordered, and the trace is cleared by rg_reset_kernel_stats; refused without the flag."""
    from paper_1807_09467_b200 import rg as rgb
    hm = random_csr(5000, rng, per_row=(2, 8), diag=2.5)
    b = rng.standard_normal(5000)
    for flags in (rgb.RG_FLAG_PROFILE, rgb.RG_FLAG_PROFILE | rgb.RG_FLAG_NO_PERSIST):
        ctx = make_ctx(hm, max_m=20, s=4, k=4, flags=flags)
        x = torch.zeros(5000, dtype=torch.float64, device=DEV)
        ctx.solve(t(b), x, m=20, variant="plain", tol=1e-9)
        ev, cnt = ctx.kernel_trace()
        assert cnt == len(ev) > 0
        starts = [e for e in ev if e[1] == 0]
        ends = [e for e in ev if e[1] == 1]
        assert len(starts) == len(ends)
        for s0 in starts:
            assert any(e[2] == s0[2] and e[0] >= s0[0] for e in ends)
        ctx.reset_kernel_stats()
        assert ctx.kernel_trace()[1] == 0
        ctx.close()
    ctx = make_ctx(hm, max_m=20, s=4, k=4)
    with pytest.raises(rgb.RgError) as e:
        ctx.kernel_trace()
    assert e.value.status == rgb.RG_E_STATE
    ctx.close()


# ------------------------------------------------------------------------------------- SELL-32-sigma
def _sell_ctx(hm, sigma, **kw):
    from paper_1807_09467_b200 import Context
    return Context(hm.n, t(hm.row_ptr), t(hm.col_idx), t(hm.val), sell_C=32, sell_sigma=sigma, **kw)


@pytest.mark.parametrize("sigma", [32, 256, 4096])
@pytest.mark.parametrize("n", [31, 1000, 4097, 70001])
def test_sell_sigma_spmv(sigma, n, rng):
    """SELL-32-sigma with row sorting inside sigma-windows (ragged rows 0..40 entries, so the order
    really changes): y = A x against the oracle at 1e-13, in the caller's row order; a values-only
    update is repacked through the same permutation."""
    hm = random_csr(n, rng, per_row=(0, 40) if n > 100 else (0, 5))
    ctx = _sell_ctx(hm, sigma)
    x = rng.standard_normal(n)
    y = torch.zeros(n, dtype=torch.float64, device=DEV)
    ctx.apply(t(x), y)
    spmv_check(hm, x, y.cpu().numpy())
    hm2 = synth.HostMatrix("csr", n, hm.row_ptr, hm.col_idx, rng.standard_normal(len(hm.val)))
    ctx.update_matrix(t(hm2.val))
    ctx.apply(t(x), y)
    spmv_check(hm2, x, y.cpu().numpy())
    ctx.close()


def test_sell_sigma_rejected_values(rng):
    from paper_1807_09467_b200 import rg as rgb
    hm = random_csr(200, rng)
    for bad in (3, 48, -1):
        with pytest.raises(rgb.RgError) as e:
            _sell_ctx(hm, bad)
        assert e.value.status == rgb.RG_E_INVAL


@pytest.mark.parametrize("variant", ["plain", "augment", "deflate", "oblique"])
def test_sell_sigma_solve_vs_oracle(variant, rng):
    """Solves with a sorted SELL-32-sigma matrix (graph path: the permutation crosses the persistent
    kernel's row ranges), including C = A W through the operator build, against the oracle."""
    from paper_1807_09467_b200 import rg as rgb
    n, m, k = 20000, 25, 6
    hm = random_csr(n, rng, per_row=(0, 24), diag=3.0)
    W = np.linalg.qr(rng.standard_normal((n, k)))[0]
    b = rng.standard_normal(n)
    ctx = _sell_ctx(hm, 512, max_m=m, max_snapshots=k, max_k=k, flags=rgb.RG_FLAG_PROFILE)
    for i in range(k):
        ctx.push_snapshot(t(W[:, i] * (k - i)))
    assert ctx.build_recycle(k)[0] == k
    x = torch.zeros(n, dtype=torch.float64, device=DEV)
    rep = ctx.solve(t(b), x, m=m, variant=variant, tol=1e-9)
    ref = oracle.solve(oracle.Matrix.from_host(hm), b, m=m, variant=variant, W=W if variant != "plain" else None,
                       tol=1e-9)
    assert rep["converged"] and ref["converged"]
    assert abs(rep["iterations"] - ref["iterations"]) <= 2
    assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])
    assert ctx.kernel_stats()["persistent_solve"]["launches"] == 0
    ctx.close()
