"""Randomised GPU-vs-oracle parity for BSR-64 SEQUENCES (seeded): random block patterns (ragged block rows,
a diagonal block in every row), 2-4 systems whose values are perturbed between systems, every variant,
recycle dimensions that cross the 8-column groups of the SpMM (k up to 20), warm starts (the start's A x0
rides in the SpMM as an extra column) and cold starts, teacher-forced like tests/test_gpu_sequence.py.
Bar: x within 1e-7 relative, iterations within +-2, sigma within max(1e-10 sigma_i, 1e-15 sigma_1).
RG_FUZZ_SEED_BASE selects other seed bases (tools/soak.sh)."""
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda"
VARIANTS = ["deflate", "augment", "oblique", "plain", "orthogonal"]


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def random_bsr(nb, rng, B=64):
    rp, ci = [0], []
    for i in range(nb):
        extra = int(rng.integers(0, min(5, nb - 1) + 1))
        cols = set(rng.choice(nb, size=extra, replace=False).tolist()) | {i}
        ci += sorted(cols)
        rp.append(len(ci))
    nnzb = len(ci)
    vals = np.empty((nnzb, B, B))   # stored column-major per block: vals[p, c, r]
    p = 0
    for i in range(nb):
        for c in ci[rp[i]:rp[i + 1]]:
            blk = rng.standard_normal((B, B)) * (0.04 if c != i else 0.1)
            if c == i:
                blk += 6.0 * np.eye(B)
            vals[p] = blk
            p += 1
    return synth.HostMatrix("bsr", nb * B, np.array(rp, np.int32), np.array(ci, np.int32), vals.reshape(-1), B)


@pytest.mark.parametrize("case", range(20))
def test_fuzz_bsr_sequence(case):
    from paper_1807_09467_b200 import Context
    base = int(os.environ.get("RG_FUZZ_SEED_BASE", "9000"))
    rng = np.random.default_rng(base + 500 + case)
    nb = int(rng.choice([1, 2, 5, 17, 40, 149, 300]))
    n = nb * 64
    variant = VARIANTS[case % len(VARIANTS)]
    k = int(rng.integers(1, 21)) if variant != "plain" else 0
    m = int(rng.integers(4, 31))
    T = int(rng.integers(2, 5))
    warm = bool(rng.integers(0, 2))
    hm = random_bsr(nb, rng)
    s_cap = max(k, 1) + int(rng.integers(0, 4))
    ctx = Context(n, t(hm.row_ptr), t(hm.col_idx), t(hm.val), fmt="bsr", block=64, max_m=m, max_snapshots=s_cap,
                  max_k=max(k, 1))
    # a window of k random directions first, so that the recycle space has its full dimension from system 1
    X = [rng.standard_normal(n) * (1.0 + i) for i in range(k)]
    for v in X:
        ctx.push_snapshot(t(v))
    val = hm.val.copy()
    xprev = None
    for step in range(1, T + 1):
        if step > 1:
            val = val * (1.0 + 0.01 * rng.uniform(-1.0, 1.0, size=val.size))
            ctx.update_matrix(t(val))
        A = synth.HostMatrix("bsr", n, hm.row_ptr, hm.col_idx, val, 64)
        b = rng.standard_normal(n)
        W = None
        if variant != "plain" and X:
            ke, sg = ctx.build_recycle(k)
            W, so, ko = oracle.recycle_basis(np.stack(X[-s_cap:], 1), k)
            assert ke == ko, (step, ke, ko)
            assert np.all(np.abs(sg[:len(so)] - so) <= np.maximum(1e-10 * so, 1e-15 * so[0]))
        x0 = xprev if (warm and xprev is not None) else None
        x = torch.zeros(n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b), x, x0=None if x0 is None else t(x0), m=m, variant=variant, tol=1e-9, max_iters=3000)
        ref = oracle.solve(oracle.Matrix.from_host(A), b, x0=x0, m=m, variant=variant, W=W, tol=1e-9, max_iters=3000)
        desc = dict(case=case, nb=nb, variant=variant, k=k, m=m, step=step, warm=warm,
                    its=(rep["iterations"], ref["iterations"]))
        assert rep["converged"] and ref["converged"], desc
        assert abs(rep["iterations"] - ref["iterations"]) <= 2, desc
        xg = x.cpu().numpy()
        assert np.linalg.norm(xg - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"]), desc
        xprev = ref["x"]
        X.append(xprev)
        ctx.push_snapshot(t(xprev))
    ctx.close()
