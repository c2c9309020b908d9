"""Distinct contexts are independent (include/rg.h: "rg_ctx ... single-owner, not thread-safe; distinct
contexts are independent"): two contexts with different matrices, variants and execution paths give bitwise
the results of running each alone — interleaved call by call on one host thread, and driven concurrently by
two host threads (ctypes releases the GIL inside the C calls, so the library really runs concurrently: its
process-wide caches, the per-context device state and the cooperative / graph launches must not interfere)."""
import threading

import numpy as np
import pytest

import synth
from test_gpu_fuzz import random_csr

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


SPECS = [  # (seed, n, variant, k, m, flags, ssor)
    (1, 6000, "deflate", 6, 30, 0, False),     # persistent path
    (2, 9000, "augment", 4, 25, 8, True),      # graph path (RG_FLAG_NO_PERSIST) + SSOR
    (3, 5000, "oblique", 5, 20, 4, False),     # classical CGS2
]


def make(spec):
    from paper_1807_09467_b200 import Context
    seed, n, variant, k, m, flags, pc = spec
    rng = np.random.default_rng(100 + seed)
    hm = random_csr(n, rng, 1, 6, diag=2.6)
    ctx = Context(n, t(hm.row_ptr), t(hm.col_idx), t(hm.val), max_m=m, max_snapshots=k + 2, max_k=k, flags=flags)
    if pc:
        ctx.set_preconditioner("ssor", 1.0)
    snaps = [rng.standard_normal(n) for _ in range(k)]
    rhs = [rng.standard_normal(n) for _ in range(3)]
    return ctx, hm, snaps, rhs


def steps(spec, ctx, hm, snaps, rhs):
    """Generator: one library call sequence per system; yields between systems (interleaving points)."""
    seed, n, variant, k, m, flags, pc = spec
    out = []
    for v in snaps:
        ctx.push_snapshot(t(v))
    yield
    val = hm.val.copy()
    for i, b in enumerate(rhs):
        if i:
            val = val * (1.0 + 0.01 * np.cos(np.arange(val.size) + i))
            ctx.update_matrix(t(val))
        ctx.build_recycle(k, deferred=True)
        yield
        x = torch.zeros(n, dtype=torch.float64, device=DEV)
        rep = ctx.solve(t(b), x, m=m, variant=variant, tol=1e-9)
        assert rep["converged"]
        out.append((rep["iterations"], x.cpu().numpy().copy()))
        ctx.push_snapshot(x)
        yield
    ctx.close()
    return out


def drain(gen):
    try:
        while True:
            next(gen)
    except StopIteration as e:
        return e.value


def solo(spec):
    return drain(steps(spec, *make(spec)))


def same(a, b):
    assert len(a) == len(b)
    for (ia, xa), (ib, xb) in zip(a, b):
        assert ia == ib
        assert np.array_equal(xa, xb)


def test_interleaved_contexts_match_solo_runs_bitwise():
    ref = [solo(s) for s in SPECS]
    gens = [steps(s, *make(s)) for s in SPECS]
    res = [None] * len(gens)
    live = list(range(len(gens)))
    while live:
        for i in list(live):
            try:
                next(gens[i])
            except StopIteration as e:
                res[i] = e.value
                live.remove(i)
    for a, b in zip(ref, res):
        same(a, b)


def test_concurrent_host_threads_match_solo_runs_bitwise():
    ref = [solo(s) for s in SPECS]
    res = [None] * len(SPECS)
    err = []

    def work(i):
        try:
            torch.cuda.set_device(0)
            for _ in range(2):   # twice: the second round meets warm process-wide caches
                res[i] = solo(SPECS[i])
        except Exception as e:  # noqa: BLE001
            err.append((i, repr(e)))

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(SPECS))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not err, err
    for a, b in zip(ref, res):
        same(a, b)


def test_create_solve_destroy_does_not_leak_device_memory():
    """60 create -> push -> build -> solve -> close cycles (graph path, persistent path, SSOR on every third):
    the free device memory returns to where it was (rg_destroy frees every buffer, graph and stream)."""
    from paper_1807_09467_b200 import Context
    rng = np.random.default_rng(5)
    hm = random_csr(4000, rng, 1, 6, diag=2.6)
    rp, ci, v = t(hm.row_ptr), t(hm.col_idx), t(hm.val)
    b = t(rng.standard_normal(hm.n))
    snap = t(rng.standard_normal(hm.n))
    x = torch.zeros(hm.n, dtype=torch.float64, device=DEV)

    def cycle(i):
        ctx = Context(hm.n, rp, ci, v, max_m=20, max_snapshots=4, max_k=2, flags=8 if i % 2 else 0)
        if i % 3 == 0:
            ctx.set_preconditioner("ssor", 1.0)
        ctx.push_snapshot(snap)
        ctx.build_recycle(2)
        assert ctx.solve(b, x, m=20, variant="deflate", tol=1e-8)["converged"]
        ctx.close()

    for i in range(6):     # warm-up: module loading, per-process caches
        cycle(i)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for i in range(60):
        cycle(i)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 <= 8 << 20, (free0, free1)   # (allocator granularity slack: 8 MiB)


def test_context_stays_usable_after_errors(rng):
    """Every error return leaves the context usable (include/rg.h: nothing aborts, throws or exits)."""
    from paper_1807_09467_b200 import Context, rg as rgb
    hm = random_csr(3000, rng, 1, 6, diag=2.6)
    ctx = Context(hm.n, t(hm.row_ptr), t(hm.col_idx), t(hm.val), max_m=20, max_snapshots=4, max_k=3)
    b = t(rng.standard_normal(hm.n))
    x = torch.zeros(hm.n, dtype=torch.float64, device=DEV)
    with pytest.raises(rgb.RgError) as e:
        ctx.build_recycle(2)                          # no snapshots yet
    assert e.value.status == rgb.RG_E_STATE
    with pytest.raises(rgb.RgError) as e:
        ctx.solve(b, x, m=21, variant="plain")        # m > max_m
    assert e.value.status == rgb.RG_E_INVAL
    with pytest.raises(rgb.RgError) as e:
        ctx.solve(b, x, m=10, variant="plain", tol=-1.0)
    assert e.value.status == rgb.RG_E_INVAL
    v = rng.standard_normal(hm.n)
    for s in (v, 2.0 * v, -v):                        # rank-1 window: k_eff = 1
        ctx.push_snapshot(t(s))
    assert ctx.build_recycle(3)[0] == 1
    r1 = ctx.solve(b, x, m=20, variant="deflate", tol=1e-9)
    assert r1["converged"]
    x1 = x.clone()
    r2 = ctx.solve(b, x, m=20, variant="deflate", tol=1e-9)   # and the same call again: bitwise the same
    assert r2["iterations"] == r1["iterations"] and torch.equal(x, x1)
    ctx.close()
