"""The Krylov basis the GPU builds, exported through the C ABI (RG_FLAG_KEEP_BASIS, rg_export
RG_EXPORT_V / _H / _B), against the invariants the north star names:
  Arnoldi relation   A V = V_{J+1} H-bar                 (plain, augment)
  GCRO relation      A V = Q B + V_{J+1} H-bar             (deflate)
  orthonormality     ||V^T V - I||_max <= 1e-12,  ||Q^T V||_max <= 1e-12
A V is formed by scipy.sparse on the host matrix and the implied next vector v_J is checked too.
Covered on every execution path the library takes (persistent cooperative kernel, CUDA graph with
DCGS2, classical CGS2) and at full BASELINE sizes (C2: persistent; C4: graph + TMA DCGS2 with the
evict-first L2 policy).  On a single-cycle solve H-bar is also compared with the oracle's (MGS2
Arnoldi, oracle.solve_basis): the Arnoldi process is unique given v_0.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda"


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _export(ctx, n, k):
    from paper_1807_09467_b200 import rg
    J = ctx.export(rg.RG_EXPORT_V, None)
    V = np.zeros(n * J)
    ctx.export(rg.RG_EXPORT_V, V)
    H = np.zeros((J + 1) * J)
    ctx.export(rg.RG_EXPORT_H, H)
    V = V.reshape(J, n).T
    H = H.reshape(J, J + 1).T
    B = Q = None
    if k:
        B = np.zeros(k * J)
        ctx.export(rg.RG_EXPORT_B, B)
        B = B.reshape(J, k).T
        Q = np.zeros(n * k)
        ctx.export(rg.RG_EXPORT_Q, Q)
        Q = Q.reshape(k, n).T
    return V, H, B, Q


def check_relation(A_s, V, H, B=None, Q=None, tol=1e-12):
    J = V.shape[1]
    assert J >= 2
    w = A_s @ V[:, J - 1] - V @ H[:J, J - 1]
    if B is not None:
        w -= Q @ B[:, J - 1]
    vJ = w / H[J, J - 1]
    V1 = np.column_stack([V, vJ])
    orth = np.max(np.abs(V1.T @ V1 - np.eye(J + 1)))
    assert orth <= tol, orth
    rhs = V @ H[:J, :J - 1]
    if B is not None:
        rhs = rhs + Q @ B[:, :J - 1]
    rel = np.linalg.norm(A_s @ V[:, :J - 1] - rhs) / sp.linalg.norm(A_s)
    assert rel <= tol * np.sqrt(J), rel
    assert np.all(np.tril(H, -2) == 0.0)
    assert np.all(np.diag(H, -1) > 0.0)
    if Q is not None:
        assert np.max(np.abs(Q.T @ V1)) <= tol
        assert np.max(np.abs(Q.T @ Q - np.eye(Q.shape[1]))) <= tol


def _ctx(hm, flags, m, k, s):
    from paper_1807_09467_b200 import Context, rg
    return Context(hm.n, _t(hm.row_ptr), _t(hm.col_idx), _t(hm.val), fmt=hm.fmt, block=hm.block, max_m=m,
                   max_snapshots=s, max_k=max(k, 1), flags=flags | rg.RG_FLAG_KEEP_BASIS)


PATHS = {"persistent": 0, "graph": 8, "cgs2": 8 | 4}   # RG_FLAG_NO_PERSIST = 8, RG_FLAG_CGS2 = 4


def _c1_case():
    cfg = synth.CONFIGS["C1"]
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    hm = seq.matrix(1, u)
    return cfg, seq, hm, u


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("variant", ["plain", "augment", "deflate"])
def test_relation_c1(path, variant):
    cfg, seq, hm, u = _c1_case()
    ctx = _ctx(hm, PATHS[path], cfg.m, cfg.k, cfg.s)
    A_s = hm.to_scipy()
    rng = np.random.default_rng(3)
    x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
    for i in range(cfg.k + 2):          # a window of solutions of nearby right-hand sides
        b = seq.rhs(1, u) * (1.0 + 0.1 * i) + rng.standard_normal(cfg.n) * 0.01
        ctx.solve(_t(b), x, m=cfg.m, variant="plain", tol=cfg.tol)
        ctx.push_snapshot(x)
    k = 0
    if variant != "plain":
        k, _ = ctx.build_recycle(cfg.k)
        assert k == cfg.k
    b = seq.rhs(1, u) * 1.37 + rng.standard_normal(cfg.n) * 0.02
    rep = ctx.solve(_t(b), x, m=cfg.m, variant=variant, tol=cfg.tol)
    assert rep["converged"]
    V, H, B, Q = _export(ctx, cfg.n, k if variant == "deflate" else 0)
    check_relation(A_s, V, H, B, Q)
    if variant == "augment":
        from paper_1807_09467_b200 import rg
        Qe = np.zeros(cfg.n * k)
        ctx.export(rg.RG_EXPORT_Q, Qe)
        Qe = Qe.reshape(k, cfg.n).T
        # augment runs Arnoldi on A from r_c with Q^T r_c = 0: v_0 is orthogonal to Q
        assert np.max(np.abs(Qe.T @ V[:, 0])) <= 1e-12
    ctx.close()


@pytest.mark.parametrize("path", list(PATHS))
def test_hessenberg_matches_oracle_single_cycle(path):
    """Plain GMRES(m) converging within one cycle: the GPU's H-bar equals the oracle's MGS2 Arnoldi
    H-bar column by column (same v_0 = b/||b||), to 1e-10 relative to ||H||."""
    rng = np.random.default_rng(11)
    n = 3000
    offs = [-61, -1, 0, 1, 60]
    diags = [rng.uniform(-1, 0, n - abs(o)) for o in offs]
    diags[2] = 6.0 + rng.random(n)
    A_s = sp.diags(diags, offs, format="csr")
    A_s.sort_indices()
    hm = synth.HostMatrix("csr", n, A_s.indptr.astype(np.int32), A_s.indices.astype(np.int32), A_s.data.copy())
    b = rng.standard_normal(n)
    ro = oracle.solve_basis(oracle.Matrix.from_host(hm), b, m=60, tol=1e-10)
    assert ro["cycles"] == 1
    ctx = _ctx(hm, PATHS[path], 60, 0, 2)
    x = torch.zeros(n, dtype=torch.float64, device=DEV)
    rep = ctx.solve(_t(b), x, m=60, variant="plain", tol=1e-10)
    assert rep["restarts"] == 0 and abs(rep["iterations"] - ro["iterations"]) <= 2
    V, H, _, _ = _export(ctx, n, 0)
    check_relation(A_s, V, H)
    J = min(V.shape[1], ro["steps"])
    Ho = ro["H"]
    assert np.max(np.abs(H[:J + 1, :J] - Ho[:J + 1, :J])) <= 1e-10 * np.linalg.norm(Ho)
    assert np.max(np.abs(V[:, :J] - ro["V"][:, :J])) <= 1e-8
    ctx.close()


@pytest.mark.parametrize("name,flags", [("C2", 0), ("C4", 0), ("C2", 8)])
@pytest.mark.parametrize("variant", ["plain", "deflate"])
def test_relation_full_size(name, flags, variant):
    """BASELINE sizes: C2 (persistent path, and the graph path), C4 (graph path, TMA DCGS2 with
    the evict-first L2 policy: the basis is larger than L2)."""
    import bench
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    from paper_1807_09467_b200 import rg
    with torch.cuda.stream(st):
        run = bench.GpuRun(cfg, variant, cfg.k, dev, st, profile=False, sell=False, sync_build=True,
                           flags=flags | rg.RG_FLAG_KEEP_BASIS)
        seq = synth.HostSequence(cfg)
        for t in range(1, 4):
            x_prev = run.x.cpu().numpy().copy()
            rep = run.step()
        torch.cuda.synchronize()
        hm = seq.matrix(3, x_prev)                 # A_3, built from x_2 exactly as the device did
        k = run.k_eff if variant == "deflate" else 0
        V, H, B, Q = _export(run.ctx, cfg.n, k)
        check_relation(hm.to_scipy(), V, H, B, Q)
        run.ctx.close()


def test_export_errors():
    from paper_1807_09467_b200 import Context, RgError, rg
    cfg, seq, hm, u = _c1_case()
    ctx = Context(hm.n, _t(hm.row_ptr), _t(hm.col_idx), _t(hm.val), max_m=30, max_snapshots=4, max_k=2)
    with pytest.raises(RgError) as e:
        ctx.export(rg.RG_EXPORT_V, None)        # flag not set
    assert e.value.status == rg.RG_E_STATE
    ctx.close()
    ctx = _ctx(hm, 0, 30, 2, 4)
    with pytest.raises(RgError):
        ctx.export(rg.RG_EXPORT_V, None)        # no solve yet
    x = torch.zeros(cfg.n, dtype=torch.float64, device=DEV)
    ctx.solve(_t(seq.rhs(1, u)), x, m=30, variant="plain", tol=1e-8)
    assert ctx.export(rg.RG_EXPORT_V, None) >= 2
    with pytest.raises(RgError):
        ctx.export(rg.RG_EXPORT_B, None)        # plain solve: no B
    ctx.close()
