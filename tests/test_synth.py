"""Input generators (synth/): closed-form pattern sizes, stencil identities, determinism.
These pin the INPUTS both sides consume (SURVEY.md §8c 'Generators')."""
import numpy as np
import pytest

import synth
from synth import CONFIGS, HostSequence, nnz_closed_form


def _check_pattern(rp, ci, n):
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == ci.shape[0]
    for i in range(0, n, max(1, n // 97)):
        row = ci[rp[i]:rp[i + 1]]
        assert np.all(np.diff(row) > 0) and row.min() >= 0 and row.max() < n


@pytest.mark.parametrize("name,N", [("C1", 32), ("C2", 24), ("C3", 20), ("C4", 9)])
def test_nnz_closed_form_and_valid_pattern(name, N):
    cfg = CONFIGS[name].reduced(N) if N != CONFIGS[name].N else CONFIGS[name]
    seq = HostSequence(cfg)
    A = seq.matrix(1, seq.initial())
    assert A.nnz == nnz_closed_form(cfg)
    _check_pattern(A.row_ptr, A.col_idx, cfg.n)


def test_full_size_closed_forms():
    assert nnz_closed_form(CONFIGS["C1"]) == 4992
    assert nnz_closed_form(CONFIGS["C2"]) == 1308672
    assert nnz_closed_form(CONFIGS["C3"]) == 9424896
    assert nnz_closed_form(CONFIGS["C4"]) == 14581760
    assert nnz_closed_form(CONFIGS["C5"]) == 223232


@pytest.mark.parametrize("name,N", [("C1", 32), ("C2", 16), ("C3", 16), ("C4", 8)])
def test_interior_rows_sum_to_inverse_dt(name, N):
    """Difference operators annihilate constants: every interior row sums to 1/dt."""
    cfg = CONFIGS[name].reduced(N)
    seq = HostSequence(cfg)
    A = seq.matrix(2, seq.initial())
    S = A.to_scipy()
    rows = np.asarray(S.sum(axis=1)).ravel()
    full = np.diff(A.row_ptr) == np.diff(A.row_ptr).max()
    d = S.diagonal()
    assert np.all(np.abs(rows[full] - 1.0 / cfg.dt) <= 1e-13 * np.abs(d[full]))


def test_zero_velocity_is_symmetric():
    L = synth.lib()
    N = 12
    h = 1.0 / (N + 1)
    n = N * N
    rp = np.empty(n + 1, np.int32)
    ci = np.empty(5 * n, np.int32)
    v = np.empty(5 * n)
    nnz = L.sy_fill5(N, 0.01 / h / h, 1 / h, 20.0, 0.0, 0.0, None, synth._ptr(rp, synth._i32p),
                     synth._ptr(ci, synth._i32p), synth._ptr(v))
    S = synth.HostMatrix("csr", n, rp, ci[:nnz], v[:nnz]).to_scipy()
    assert abs(S - S.T).max() == 0.0


def test_upwind_direction_follows_velocity_sign():
    """C2: beta = u_{t-1}(1,1) per node; the W neighbour carries the convection only if u > 0."""
    cfg = CONFIGS["C2"].reduced(8)
    seq = HostSequence(cfg)
    u = np.linspace(-1, 1, cfg.n)
    S = seq.matrix(2, u).to_scipy().toarray()
    sc = seq.scalars()
    cd, ih = sc["cd"], sc["ih"]
    r = 2 * 8 + 3                     # interior node with u < 0
    assert u[r] < 0 and S[r, r - 1] == -cd and S[r, r + 1] == -(cd + (-u[r]) * ih)
    r2 = 5 * 8 + 3
    assert u[r2] > 0 and S[r2, r2 - 1] == -(cd + u[r2] * ih) and S[r2, r2 + 1] == -cd


def test_deterministic_and_seeded():
    a = HostSequence(CONFIGS["C1"]).initial()
    b = HostSequence(CONFIGS["C1"]).initial()
    assert np.array_equal(a, b) and a.max() > 0.1
    c = HostSequence(CONFIGS["C3"].reduced(32)).initial()
    assert not np.array_equal(a, c[: a.shape[0]])


def test_c5_blocks_and_perturbation():
    cfg = CONFIGS["C5"].reduced(3)
    seq = HostSequence(cfg)
    A1 = seq.matrix(1)
    A3 = seq.matrix(3)
    assert A1.col_idx.shape[0] == nnz_closed_form(cfg) == 27 + 6 * 9 * 2
    ratio = A3.val / A1.val
    assert np.all(np.abs(ratio - 1) <= 0.0201 + 1e-12) and np.abs(ratio - 1).max() > 0.005
    B = cfg.B
    diag_blk = A1.val[: B * B].reshape(B, B)   # block 0 of row 0 is the diagonal block (no -z/-y/-x)
    assert abs(np.mean(np.diag(diag_blk)) - 100) < 1.0
    b = seq.rhs(1, None)
    assert abs(b.mean()) < 0.1 and abs(b.std() - 1) < 0.1


@pytest.mark.gpu
@pytest.mark.parametrize("nval,off", [(1, 0), (7, 0), (7, 1), (100003, 0), (100003, 1), (2 * 148 * 16 * 256 * 4 + 5, 0)])
def test_c5_perturb_device_matches_host(nval, off):
    """The device perturbation (16-byte vectorised, 4 pairs in flight; scalar path when the buffer is
    not 16-byte aligned; odd tail) is bit-identical to the host C loop (R10: A_t = A_{t-1} o (1+0.01 xi))."""
    import ctypes
    torch = pytest.importorskip("torch")
    L, C = synth.lib(), synth.culib()
    rng = np.random.default_rng(nval)
    v = rng.standard_normal(nval + off)
    ref = v[off:].copy()
    L.sy_c5_perturb(nval, 1234, 3, ref.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    d = torch.from_numpy(v).cuda()
    assert C.syd_c5_perturb(nval, 1234, 3, ctypes.c_void_p(d.data_ptr() + 8 * off), None) == 0
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy()[off:], ref)


@pytest.mark.gpu
@pytest.mark.parametrize("name,t", [("C1", 3), ("C2", 2), ("C4", 5), ("C5", 3)])
def test_device_stencil_and_rhs_match_host_full_size(name, t):
    """The device generator bench.py times (syd_fill5_values / syd_fill7_values / syd_rhs /
    syd_c5_values + perturbation / syd_normal_vec) writes bit-identical A_t and b_t to the host
    generator the oracle consumes, at the configs' FULL sizes (C2: velocity u_{t-1}(1,1) per node;
    C1 / C4: time-dependent constant velocity; C5: base blocks and the cumulative 1 % perturbation)."""
    torch = pytest.importorskip("torch")
    cfg = CONFIGS[name]
    seq = HostSequence(cfg)
    rng = np.random.default_rng(7)
    u = seq.initial() + 0.05 * rng.standard_normal(cfg.n)   # any x_{t-1}, signs of both kinds
    gen = synth.DeviceSequence(cfg, "cuda")
    ud = torch.from_numpy(u).cuda()
    gen.fill(1, ud)
    gen.fill(t, ud)
    torch.cuda.synchronize()
    A = seq.matrix(t, u)
    assert np.array_equal(gen.row_ptr.cpu().numpy(), A.row_ptr)
    assert np.array_equal(gen.col_idx.cpu().numpy(), A.col_idx)
    assert np.array_equal(gen.val.cpu().numpy(), A.val)
    assert np.array_equal(gen.b.cpu().numpy(), seq.rhs(t, u))
