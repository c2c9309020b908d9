import sys, numpy as np, torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle, synth
from test_gpu_parity import random_csr, make_ctx, t
rng = np.random.default_rng(1)
n, k = 200, 4
hm = random_csr(n, rng, per_row=(2, 8), diag=2.2)
W = np.linalg.qr(rng.standard_normal((n, k)))[0]
ctx = make_ctx(hm, max_m=10, s=k, k=k)
for i in range(k):
    ctx.push_snapshot(t(W[:, i] * (k - i)))
ke, sig = ctx.build_recycle(k)
print("ke", ke, "sig", sig[:k])
Wg = np.zeros((k, n)); ctx.export(0, Wg); Wg = Wg.T
print("WtW", np.round(Wg.T @ Wg, 6))
print("span err", np.linalg.norm(Wg @ Wg.T - W @ W.T, 2))
b = rng.standard_normal(n)
x = torch.zeros(n, dtype=torch.float64, device='cuda')
try:
    rep = ctx.solve(t(b), x, m=10, variant='deflate', tol=1e-8, history_cap=100)
    print(rep)
except Exception as e:
    print("ERR", e)
