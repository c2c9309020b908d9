"""Randomised GPU-vs-oracle parity for CSR / SELL SEQUENCES with option interplay (seeded): values-only
matrix updates between systems with the SSOR preconditioner set (its colour-ordered copies, incl. the
pre-scaled couplings of the fused forward sweep, must follow the values), largest / smallest recycle modes,
host or device buffers for b / x / snapshots, window eviction, every variant and execution path.
Teacher-forced like tests/test_gpu_sequence.py; bar: x within 1e-7 relative, iterations within +-2.
RG_FUZZ_SEED_BASE selects other seed bases (tools/soak.sh)."""
import os

import numpy as np
import pytest

import oracle
import synth
from coloring import greedy_colors
from test_gpu_fuzz import random_csr

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda"
VARIANTS = ["deflate", "augment", "oblique", "orthogonal", "plain"]


def t(a, host=False):
    x = torch.from_numpy(np.ascontiguousarray(a))
    return x if host else x.to(DEV)


@pytest.mark.parametrize("case", range(20))
def test_fuzz_csr_sequence(case):
    from paper_1807_09467_b200 import Context, rg as rgb
    base = int(os.environ.get("RG_FUZZ_SEED_BASE", "9000"))
    rng = np.random.default_rng(base + 700 + case)
    n = int(rng.choice([65, 500, 4097, 30000]))
    variant = VARIANTS[case % len(VARIANTS)]
    k = int(rng.integers(1, 13)) if variant != "plain" else 0
    m = int(rng.integers(5, 41))
    T = int(rng.integers(2, 5))
    sell = bool(rng.integers(0, 2))
    pc = bool(rng.integers(0, 2))
    omega = float(rng.choice([1.0, 1.2]))
    modes = "smallest" if (variant != "plain" and rng.integers(0, 3) == 0) else "largest"
    host = bool(rng.integers(0, 3) == 0)
    flags = int(rng.choice([0, 0, rgb.RG_FLAG_NO_PERSIST, rgb.RG_FLAG_CGS2]))
    hm = random_csr(n, rng, 1, 6, diag=float(rng.uniform(2.0, 3.0)))
    s_cap = max(k, 1) + int(rng.integers(0, 3))
    ctx = Context(n, t(hm.row_ptr), t(hm.col_idx), t(hm.val), sell_C=32 if sell else 0, max_m=m, max_snapshots=s_cap,
                  max_k=max(k, 1), flags=flags)
    order = None
    if pc:
        col = greedy_colors(n, hm.row_ptr, hm.col_idx)
        ctx.set_preconditioner("ssor", omega, colors=col)
        order = oracle.ssor_order(col)
    # graded window: the smallest modes are well separated from rounding
    X = [rng.standard_normal(n) * 2.0 ** (-i) for i in range(k)]
    for v in X:
        ctx.push_snapshot(t(v, host))
    val = hm.val.copy()
    for step in range(1, T + 1):
        if step > 1:
            val = val * (1.0 + 0.02 * rng.uniform(-1.0, 1.0, size=val.size))
            ctx.update_matrix(t(val, host))
        A = synth.HostMatrix("csr", n, hm.row_ptr, hm.col_idx, val)
        b = rng.standard_normal(n)
        W = None
        if variant != "plain" and X:
            ke, _ = ctx.build_recycle(k, modes=modes)
            W, _, ko = oracle.recycle_basis(np.stack(X[-s_cap:], 1), k, modes=modes)
            assert ke == ko, (step, ke, ko)
        x = torch.zeros(n, dtype=torch.float64) if host else torch.zeros(n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b, host), x, m=m, variant=variant, tol=1e-9, max_iters=4000)
        ref = oracle.solve(oracle.Matrix.from_host(A), b, m=m, variant=variant, W=W, tol=1e-9, max_iters=4000,
                           precond=None if order is None else (order, omega))
        desc = dict(case=case, n=n, variant=variant, k=k, m=m, step=step, sell=sell, pc=pc, modes=modes, host=host,
                    flags=flags, its=(rep["iterations"], ref["iterations"]))
        assert rep["converged"] == ref["converged"], desc
        if ref["converged"]:
            assert abs(rep["iterations"] - ref["iterations"]) <= 2, desc
            xg = x.cpu().numpy()
            assert np.linalg.norm(xg - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"]), desc
        u = ref["x"]
        X.append(u)
        ctx.push_snapshot(t(u, host))
    ctx.close()
