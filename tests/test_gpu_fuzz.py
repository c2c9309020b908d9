"""Randomised GPU-vs-oracle parity over the option space (seeded, reproducible): matrix size and
sparsity (ragged rows, n from 1 to 20,000, so single- and multi-CTA persistent solves occur), restart
length, recycle dimension, variant, SELL packing (sigma 1 / 32 / 256), SSOR, nonzero x0, and the execution path (persistent,
CUDA graph, classical CGS2).
Bar as in test_gpu_parity: x within 1e-7 relative, iterations within +-2, true residual <= tol."""
import os

import numpy as np
import pytest

import oracle
import synth
from coloring import greedy_colors

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda"
VARIANTS = ["plain", "augment", "deflate", "oblique", "orthogonal"]


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def random_csr(n, rng, lo, hi, diag):
    rp, ci, v = [0], [], []
    for i in range(n):
        nr = int(rng.integers(lo, hi + 1))
        cols = set(rng.choice(n, size=min(nr, n), replace=False).tolist()) | {i}
        for c in sorted(cols):
            ci.append(c)
            v.append(diag if c == i else rng.standard_normal() / np.sqrt(max(nr, 1)))
        rp.append(len(ci))
    return synth.HostMatrix("csr", n, np.array(rp, np.int32), np.array(ci, np.int32), np.array(v))


@pytest.mark.parametrize("case", range(60))
def test_fuzz_case(case):
    from paper_1807_09467_b200 import Context
    # RG_FUZZ_SEED_BASE (soak runs, tools/soak.sh): other seed bases draw new cases; they also draw
    # n = 150,001 (every TMA pass on its full 148-CTA grid with a ragged last tile)
    base = int(os.environ.get("RG_FUZZ_SEED_BASE", "9000"))
    rng = np.random.default_rng(base + case)
    sizes = [1, 7, 63, 64, 65, 500, 4096, 4097, 20000] + ([150001] if base != 9000 else [])
    n = int(rng.choice(sizes))
    m = int(rng.integers(1, 41 if base == 9000 else 101))   # soak runs: m > 64 forces the graph path
    variant = VARIANTS[case % len(VARIANTS)] if n > 1 else "plain"
    kmax = 8 if base == 9000 else 24   # soak runs also reach the k > 16 operator-build paths
    k = int(rng.integers(1, min(kmax, max(n - 1, 1)) + 1)) if variant != "plain" else 0
    sell = bool(rng.integers(0, 2))
    pc = bool(rng.integers(0, 3) == 0)
    omega = float(rng.choice([1.0, 1.3]))
    hm = random_csr(n, rng, 1, 6, diag=float(rng.uniform(1.8, 3.0)))
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n) * 0.1 if rng.integers(0, 2) else None
    from paper_1807_09467_b200 import rg as rgb
    flags = int(rng.choice([0, 0, rgb.RG_FLAG_NO_PERSIST, rgb.RG_FLAG_CGS2]))  # persistent / graph / classical CGS2
    if base != 9000:  # soak runs: also the host-driven loop, profiling and basis-keeping builds of each path
        flags |= int(np.random.default_rng(base + 31337 + case).choice(
            [0, 0, rgb.RG_FLAG_NO_GRAPH, rgb.RG_FLAG_PROFILE, rgb.RG_FLAG_KEEP_BASIS,
             rgb.RG_FLAG_NO_GRAPH | rgb.RG_FLAG_NO_PERSIST, rgb.RG_FLAG_PROFILE | rgb.RG_FLAG_KEEP_BASIS]))
    # SELL-32-sigma row sorting (own generator: the main draw sequence of the cases stays as it was)
    sigma = int(np.random.default_rng(base - 1300 + case).choice([1, 32, 256])) if sell else 1
    ctx = Context(n, t(hm.row_ptr), t(hm.col_idx), t(hm.val), sell_C=32 if sell else 0, max_m=max(m, 2),
                  max_snapshots=max(k, 1), max_k=max(k, 1), flags=flags, sell_sigma=sigma)
    W = None
    if k:
        W = np.linalg.qr(rng.standard_normal((n, k)))[0]
        for i in range(k):
            ctx.push_snapshot(t(W[:, i] * (k - i)))
        assert ctx.build_recycle(k)[0] == k
    order = None
    if pc:
        col = greedy_colors(n, hm.row_ptr, hm.col_idx)
        ctx.set_preconditioner("ssor", omega, colors=col)
        order = oracle.ssor_order(col)
    x = torch.zeros(n, dtype=torch.float64, device=DEV)
    rep = ctx.solve(t(b), x, x0=None if x0 is None else t(x0), m=m, variant=variant, tol=1e-9, max_iters=5000)
    ref = oracle.solve(oracle.Matrix.from_host(hm), b, x0=x0, m=m, variant=variant, W=W, tol=1e-9,
                       max_iters=5000, precond=None if order is None else (order, omega))
    desc = dict(n=n, m=m, k=k, variant=variant, sell=sell, sigma=sigma, pc=pc, x0=x0 is not None, flags=flags,
                its=(rep["iterations"], ref["iterations"]))
    assert rep["converged"] == ref["converged"], desc
    if ref["converged"]:
        assert abs(rep["iterations"] - ref["iterations"]) <= 2, desc
        xg = x.cpu().numpy()
        assert np.linalg.norm(xg - ref["x"]) <= 1e-7 * max(np.linalg.norm(ref["x"]), 1e-300), desc
        r = b - oracle.spmv(oracle.Matrix.from_host(hm), xg)
        assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(b) * 1.001, desc
    ctx.close()
