"""Teacher-forced sequence parity: for each system the oracle's x_{t-1}
builds A_t, b_t and is the snapshot pushed to BOTH sides; the GPU builds its own recycle space
(two-pass Gram-Jacobi SVD) and solves; the oracle builds its own (one-sided Jacobi) and solves.
Compared per system: singular values, solution, iteration count."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def run(cfg, variant, T, k=None):
    from paper_1807_09467_b200 import Context
    k = k or cfg.k
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    A1 = seq.matrix(1, u)
    ctx = Context(cfg.n, t(A1.row_ptr), t(A1.col_idx), t(A1.val), fmt=A1.fmt, block=A1.block,
                  sell_C=32 if cfg.fmt == "sell" else 0, max_m=cfg.m, max_snapshots=cfg.s, max_k=k)
    X = []
    rows = []
    for step in range(1, T + 1):
        A = seq.matrix(step, u)
        b = seq.rhs(step, u)
        ctx.update_matrix(t(A.val))
        W = None
        sg = so = None
        if variant != "plain" and X:
            ke, sg = ctx.build_recycle(k)
            W, so, ko = oracle.recycle_basis(np.stack(X[-cfg.s:], 1), k)
            assert ke == ko
        x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b), x, m=cfg.m, variant=variant, tol=cfg.tol)
        ref = oracle.solve(oracle.Matrix.from_host(A), b, m=cfg.m, variant=variant, W=W, tol=cfg.tol)
        xg = x.cpu().numpy()
        rows.append((step, rep["iterations"], ref["iterations"],
                     np.linalg.norm(xg - ref["x"]) / np.linalg.norm(ref["x"])))
        assert rep["converged"] and ref["converged"], rows[-1]
        assert abs(rep["iterations"] - ref["iterations"]) <= 2, rows
        assert rows[-1][3] <= 1e-7, rows
        if sg is not None:
            s = len(so)
            assert np.all(np.abs(sg[:s] - so) <= np.maximum(1e-10 * so, 1e-15 * so[0])), (sg[:s], so)
        u = ref["x"]
        X.append(u)
        ctx.push_snapshot(t(u))
    ctx.close()
    return rows


@pytest.mark.parametrize("variant", ["plain", "augment", "deflate", "oblique", "orthogonal"])
def test_c1_full_sequence(variant):
    run(synth.CONFIGS["C1"], variant, 10)


@pytest.mark.parametrize("variant", ["augment", "deflate", "oblique", "orthogonal"])
def test_c2_reduced(variant):
    run(synth.CONFIGS["C2"].reduced(96), variant, 6)


def test_c3_reduced_sell_deflate():
    run(synth.CONFIGS["C3"].reduced(96), "deflate", 5)


@pytest.mark.parametrize("variant", ["augment", "deflate", "oblique"])
def test_c4_reduced(variant):
    run(synth.CONFIGS["C4"].reduced(20), variant, 5, k=8)


@pytest.mark.parametrize("variant", ["deflate", "oblique"])
def test_c5_reduced_bsr(variant):
    run(synth.CONFIGS["C5"].reduced(3), variant, 5)


@pytest.mark.parametrize("variant,host", [("augment", False), ("deflate", False), ("oblique", False),
                                          ("deflate", True)])
def test_c5_warm_start_fused_start_residual(variant, host):
    """BSR-64 graph path with a NONZERO initial guess x0 = x_{t-1}: the solve-start product A x0
    rides along as an extra column of the C = A W SpMM (SM_RES_Y start) — every recycled solve
    must take that path (kernel statistics) and still match the oracle started from the same x0.
    host=True: b, x0 and x_out are HOST arrays (x0 is copied in before the SpMM reads it)."""
    from paper_1807_09467_b200 import Context, rg as rgb
    cfg = synth.CONFIGS["C5"].reduced(3)
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    A1 = seq.matrix(1, u)
    ctx = Context(cfg.n, t(A1.row_ptr), t(A1.col_idx), t(A1.val), fmt="bsr", block=A1.block, max_m=cfg.m,
                  max_snapshots=cfg.s, max_k=cfg.k, flags=rgb.RG_FLAG_PROFILE)
    X, fused = [], 0
    for step in range(1, 5):
        A = seq.matrix(step, u)
        b = seq.rhs(step, u)
        ctx.update_matrix(t(A.val))
        W = None
        if X:
            ke, _ = ctx.build_recycle(cfg.k)
            W, _, ko = oracle.recycle_basis(np.stack(X[-cfg.s:], 1), cfg.k)
            assert ke == ko
            fused += 1
        if host:
            x = np.zeros(cfg.n)
            rep = ctx.solve(np.ascontiguousarray(b), x, x0=np.ascontiguousarray(u), m=cfg.m, variant=variant,
                            tol=cfg.tol)
            xg = x
        else:
            x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
            rep = ctx.solve(t(b), x, x0=t(u), m=cfg.m, variant=variant, tol=cfg.tol)
            xg = x.cpu().numpy()
        ref = oracle.solve(oracle.Matrix.from_host(A), b, x0=u, m=cfg.m, variant=variant, W=W, tol=cfg.tol)
        assert rep["converged"] and ref["converged"]
        assert abs(rep["iterations"] - ref["iterations"]) <= 2, (step, rep["iterations"], ref["iterations"])
        assert np.linalg.norm(xg - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])
        u = ref["x"]
        X.append(u)
        ctx.push_snapshot(t(u))
    st = ctx.kernel_stats()
    assert st["res_from_ax"]["launches"] == fused, st["res_from_ax"]
    ctx.close()


@pytest.mark.parametrize("variant", ["oblique", "orthogonal"])
def test_c3_reduced_sell_galerkin(variant):
    run(synth.CONFIGS["C3"].reduced(96), variant, 5)


def run_schedule(cfg, variant, T, ell=1, modes="largest", k=None):
    """Algorithm 1 with SVD interval ell (P:551 'if (i mod l) = 0') and mode selection: the recycle
    space is rebuilt only before systems t with (t-1) mod ell == 0 and kept in between."""
    from paper_1807_09467_b200 import Context
    k = k or cfg.k
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    A1 = seq.matrix(1, u)
    ctx = Context(cfg.n, t(A1.row_ptr), t(A1.col_idx), t(A1.val), max_m=cfg.m, max_snapshots=cfg.s, max_k=k)
    X, W = [], None
    its = []
    for step in range(1, T + 1):
        A = seq.matrix(step, u)
        b = seq.rhs(step, u)
        ctx.update_matrix(t(A.val))
        if X and (step - 1) % ell == 0:
            ke, sg = ctx.build_recycle(k, modes)
            W, so, ko = oracle.recycle_basis(np.stack(X[-cfg.s:], 1), k, modes)
            assert ke == ko
        x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b), x, m=cfg.m, variant=variant, tol=cfg.tol)
        ref = oracle.solve(oracle.Matrix.from_host(A), b, m=cfg.m, variant=variant, W=W, tol=cfg.tol)
        assert rep["converged"] and ref["converged"]
        assert abs(rep["iterations"] - ref["iterations"]) <= 2, (step, rep["iterations"], ref["iterations"])
        assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])
        its.append(rep["iterations"])
        u = ref["x"]
        X.append(u)
        ctx.push_snapshot(t(u))
    ctx.close()
    return its


@pytest.mark.parametrize("ell", [3])
def test_c1_svd_interval(ell):
    run_schedule(synth.CONFIGS["C1"], "deflate", 10, ell=ell)


@pytest.mark.parametrize("variant", ["deflate", "augment"])
def test_c1_smallest_modes(variant):
    run_schedule(synth.CONFIGS["C1"], variant, 8, modes="smallest", k=3)
