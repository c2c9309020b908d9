"""GPU parity of the multicolour SSOR right preconditioner (R18)
against the oracle's SSOR in the same row order (tests/coloring.py gives both sides the colours).

Tolerances: M^{-1} x  <= 1e-13 relative (same sweep arithmetic, different summation order only
inside a row); solves as in test_gpu_parity (x <= 1e-7 relative, iterations +-2)."""
import numpy as np
import pytest

import oracle
import synth
from coloring import greedy_colors

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def random_csr(n, rng, per_row=(2, 8), diag=2.2):
    rp, ci, v = [0], [], []
    for i in range(n):
        nr = rng.integers(per_row[0], per_row[1] + 1)
        cols = set(rng.choice(n, size=min(nr, n), replace=False).tolist()) | {i}
        for c in sorted(cols):
            ci.append(c)
            v.append(diag if c == i else rng.standard_normal() / np.sqrt(max(nr, 1)))
        rp.append(len(ci))
    return synth.HostMatrix("csr", n, np.array(rp, np.int32), np.array(ci, np.int32), np.array(v))


def ctx_for(hm, max_m=64, s=16, k=8, sell=False, flags=0):
    from paper_1807_09467_b200 import Context
    return Context(hm.n, t(hm.row_ptr), t(hm.col_idx), t(hm.val), sell_C=32 if sell else 0,
                   max_m=max_m, max_snapshots=s, max_k=k, flags=flags)


@pytest.mark.parametrize("omega", [1.0, 1.4])
@pytest.mark.parametrize("n", [1, 37, 2000])
def test_ssor_apply_vs_oracle(rng, n, omega):
    hm = random_csr(n, rng)
    col = greedy_colors(n, hm.row_ptr, hm.col_idx)
    ctx = ctx_for(hm)
    nc = ctx.set_preconditioner("ssor", omega, colors=col)
    assert nc == col.max() + 1
    x = rng.standard_normal(n)
    y = torch.zeros(n, dtype=torch.float64, device=DEV)
    ctx.apply_preconditioner(t(x), y)
    ref = oracle.ssor(oracle.Matrix.from_host(hm), oracle.ssor_order(col), omega, x)
    assert np.linalg.norm(y.cpu().numpy() - ref) <= 1e-13 * np.linalg.norm(ref)
    # the library's own greedy colouring is the same algorithm: same colours, same result
    assert ctx.set_preconditioner("ssor", omega) == nc
    y2 = torch.zeros(n, dtype=torch.float64, device=DEV)
    ctx.apply_preconditioner(t(x), y2)
    assert torch.equal(y, y2)


@pytest.mark.parametrize("variant", ["plain", "augment", "deflate", "oblique", "orthogonal"])
def test_preconditioned_solve_vs_oracle(rng, variant):
    n, m, k = 1500, 20, 6
    hm = random_csr(n, rng, diag=1.6)
    col = greedy_colors(n, hm.row_ptr, hm.col_idx)
    W = np.linalg.qr(rng.standard_normal((n, k)))[0]
    b = rng.standard_normal(n)
    ctx = ctx_for(hm, max_m=m, s=k, k=k)
    for i in range(k):
        ctx.push_snapshot(t(W[:, i] * (k - i)))
    assert ctx.build_recycle(k)[0] == k
    ctx.set_preconditioner("ssor", 1.0, colors=col)
    x = torch.zeros(n, dtype=torch.float64, device=DEV)
    rep = ctx.solve(t(b), x, m=m, variant=variant, tol=1e-9, history_cap=2000)
    ref = oracle.solve(oracle.Matrix.from_host(hm), b, m=m, variant=variant, W=W if variant != "plain" else None,
                       tol=1e-9, precond=(oracle.ssor_order(col), 1.0))
    assert rep["converged"] and ref["converged"]
    assert abs(rep["iterations"] - ref["iterations"]) <= 2, (rep["iterations"], ref["iterations"])
    xg = x.cpu().numpy()
    assert np.linalg.norm(xg - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])
    r = b - oracle.spmv(oracle.Matrix.from_host(hm), xg)
    assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(b) * 1.0001
    # fewer iterations than unpreconditioned
    ctx.set_preconditioner(None)
    x2 = torch.zeros(n, dtype=torch.float64, device=DEV)
    rep0 = ctx.solve(t(b), x2, m=m, variant=variant, tol=1e-9)
    assert rep["iterations"] < rep0["iterations"]


@pytest.mark.parametrize("flags", [0, 4])  # DCGS2 and classical CGS2 (RG_FLAG_CGS2)
def test_cgs2_and_dcgs2_preconditioned_agree(rng, flags):
    n = 3000
    hm = random_csr(n, rng, diag=1.5)
    b = rng.standard_normal(n)
    col = greedy_colors(n, hm.row_ptr, hm.col_idx)
    ctx = ctx_for(hm, max_m=15, flags=flags)
    ctx.set_preconditioner("ssor", 1.2, colors=col)
    x = torch.zeros(n, dtype=torch.float64, device=DEV)
    rep = ctx.solve(t(b), x, m=15, tol=1e-10)
    ref = oracle.solve(oracle.Matrix.from_host(hm), b, m=15, tol=1e-10, precond=(oracle.ssor_order(col), 1.2))
    assert rep["converged"] and abs(rep["iterations"] - ref["iterations"]) <= 2
    assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-8 * np.linalg.norm(ref["x"])


def run_seq(cfg, variant, T, k=None, sell=False, omega=1.0):
    from paper_1807_09467_b200 import Context
    k = k or cfg.k
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    A1 = seq.matrix(1, u)
    col = greedy_colors(A1.n, A1.row_ptr, A1.col_idx)
    order = oracle.ssor_order(col)
    ctx = Context(cfg.n, t(A1.row_ptr), t(A1.col_idx), t(A1.val), sell_C=32 if sell else 0, max_m=cfg.m,
                  max_snapshots=cfg.s, max_k=k)
    ctx.set_preconditioner("ssor", omega, colors=col)
    X, its = [], []
    for step in range(1, T + 1):
        A = seq.matrix(step, u)
        b = seq.rhs(step, u)
        ctx.update_matrix(t(A.val))
        W = None
        if variant != "plain" and X:
            ke, _ = ctx.build_recycle(k)
            W, _, ko = oracle.recycle_basis(np.stack(X[-cfg.s:], 1), k)
            assert ke == ko
        x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b), x, m=cfg.m, variant=variant, tol=cfg.tol)
        ref = oracle.solve(oracle.Matrix.from_host(A), b, m=cfg.m, variant=variant, W=W, tol=cfg.tol,
                           precond=(order, omega))
        assert rep["converged"] and ref["converged"]
        assert abs(rep["iterations"] - ref["iterations"]) <= 2, (step, rep["iterations"], ref["iterations"])
        assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])
        its.append(rep["iterations"])
        u = ref["x"]
        X.append(u)
        ctx.push_snapshot(t(u))
    ctx.close()
    return its


@pytest.mark.parametrize("variant", ["plain", "deflate", "oblique"])
def test_c1_sequence_ssor(variant):
    run_seq(synth.CONFIGS["C1"], variant, 8)


def test_c2_reduced_ssor_deflate():
    run_seq(synth.CONFIGS["C2"].reduced(96), "deflate", 5)


def test_c3_reduced_sell_ssor_augment():
    run_seq(synth.CONFIGS["C3"].reduced(96), "augment", 4, sell=True)


def test_c4_reduced_ssor_oblique():
    run_seq(synth.CONFIGS["C4"].reduced(16), "oblique", 4, k=8)


def test_invalid_inputs_and_pattern_change(rng):
    from paper_1807_09467_b200 import rg as rgb
    hm = random_csr(200, rng)
    ctx = ctx_for(hm)
    bad = np.zeros(200, np.int32)                    # everything one colour: coupled rows clash
    with pytest.raises(rgb.RgError) as e:
        ctx.set_preconditioner("ssor", 1.0, colors=bad)
    assert e.value.status == rgb.RG_E_INVAL
    with pytest.raises(rgb.RgError):
        ctx.set_preconditioner("ssor", 2.0)          # omega outside (0, 2)
    y = torch.zeros(200, dtype=torch.float64, device=DEV)
    with pytest.raises(rgb.RgError) as e:
        ctx.apply_preconditioner(t(np.ones(200)), y)
    assert e.value.status == rgb.RG_E_STATE
    # a row without a stored diagonal entry
    rp = np.array([0, 1, 2], np.int32); ci = np.array([1, 0], np.int32)
    h2 = synth.HostMatrix("csr", 2, rp, ci, np.array([1.0, 1.0]))
    c2 = ctx_for(h2)
    with pytest.raises(rgb.RgError):
        c2.set_preconditioner("ssor", 1.0)
    # pattern change drops the preconditioner; values-only keeps it
    ctx.set_preconditioner("ssor", 1.0)
    ctx.update_matrix(t(hm.val * 1.5))
    ctx.apply_preconditioner(t(np.ones(200)), y)
    h3 = random_csr(200, rng)
    ctx.update_matrix(t(h3.val), t(h3.row_ptr), t(h3.col_idx))
    with pytest.raises(rgb.RgError) as e:
        ctx.apply_preconditioner(t(np.ones(200)), y)
    assert e.value.status == rgb.RG_E_STATE


@pytest.mark.parametrize("variant", ["plain", "deflate", "oblique"])
def test_persistent_and_graph_paths_agree_preconditioned(rng, variant):
    """SSOR sweeps inside the cooperative solve (neighbour-synchronised colour sweeps) and the
    per-colour launches of the graph path give the same iterates."""
    from paper_1807_09467_b200 import rg as rgb
    cfg = synth.CONFIGS["C2"].reduced(160)
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    hm = seq.matrix(1, u)
    b = seq.rhs(1, u)
    snaps = [rng.standard_normal(cfg.n) for _ in range(4)]
    out = []
    for flags in (0, rgb.RG_FLAG_NO_PERSIST):
        ctx = ctx_for(hm, max_m=cfg.m, s=8, k=4, flags=flags)
        ctx.set_preconditioner("ssor", 1.1)
        for v in snaps:
            ctx.push_snapshot(t(v))
        ctx.build_recycle(4)
        x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b), x, m=cfg.m, variant=variant, history_cap=1000)
        out.append((rep, x.cpu().numpy()))
        ctx.close()
    (r0, x0), (r1, x1) = out
    assert r0["converged"] and r1["converged"]
    assert abs(r0["iterations"] - r1["iterations"]) <= 1
    assert np.linalg.norm(x0 - x1) <= 1e-9 * np.linalg.norm(x1)


def grid5(N, rng):
    """5-point stencil on an N x N grid with random couplings: exactly 2 colours (red-black)."""
    n = N * N
    rp, ci, v = [0], [], []
    for j in range(N):
        for i in range(N):
            r = j * N + i
            for (di, dj) in ((0, -1), (-1, 0), (0, 0), (1, 0), (0, 1)):
                ii, jj = i + di, j + dj
                if 0 <= ii < N and 0 <= jj < N:
                    ci.append(jj * N + ii)
                    v.append(4.5 if (di, dj) == (0, 0) else -1.0 + 0.3 * rng.standard_normal())
            rp.append(len(ci))
    return synth.HostMatrix("csr", n, np.array(rp, np.int32), np.array(ci, np.int32), np.array(v))


@pytest.mark.parametrize("omega", [1.0, 1.3])
def test_ssor_two_colours_fused_forward_sweep_and_value_update(rng, omega):
    """2 colours: the forward sweeps of colours 0 and 1 run as ONE launch (colour-0 values formed on the
    fly, couplings pre-scaled by 1 / a_jj when the values are gathered); n spans many CTAs and a ragged
    last one.  A values-only update must re-gather the pre-scaled couplings."""
    hm = grid5(301, rng)
    col = greedy_colors(hm.n, hm.row_ptr, hm.col_idx)
    assert col.max() == 1
    ctx = ctx_for(hm)
    assert ctx.set_preconditioner("ssor", omega, colors=col) == 2
    order = oracle.ssor_order(col)
    for rep in range(2):
        x = rng.standard_normal(hm.n)
        y = torch.zeros(hm.n, dtype=torch.float64, device=DEV)
        ctx.apply_preconditioner(t(x), y)
        ref = oracle.ssor(oracle.Matrix.from_host(hm), order, omega, x)
        assert np.linalg.norm(y.cpu().numpy() - ref) <= 1e-13 * np.linalg.norm(ref)
        assert np.max(np.abs(y.cpu().numpy() - ref)) <= 1e-12 * np.max(np.abs(ref))
        hm = synth.HostMatrix("csr", hm.n, hm.row_ptr, hm.col_idx, hm.val * (1.0 + 0.2 * rng.random(hm.val.size)))
        ctx.update_matrix(t(hm.val))   # values only: Lv, Uv, 1 / a_rr and the pre-scaled Lv1 follow
    ctx.close()


def test_ssor_one_colour_diagonal_matrix(rng):
    """A diagonal matrix has one colour: a single forward launch, no backward sweep; M^{-1} = w(2-w) D^{-1}."""
    n, omega = 5000, 1.2
    d = 1.0 + rng.random(n)
    hm = synth.HostMatrix("csr", n, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), d)
    ctx = ctx_for(hm)
    assert ctx.set_preconditioner("ssor", omega) == 1
    x = rng.standard_normal(n)
    y = torch.zeros(n, dtype=torch.float64, device=DEV)
    ctx.apply_preconditioner(t(x), y)
    np.testing.assert_allclose(y.cpu().numpy(), omega * (2.0 - omega) * x / d, rtol=1e-14, atol=0)
    ctx.close()
