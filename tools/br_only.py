"""build_recycle in isolation (C2 sizes): python tools/br_only.py [calls]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1807_09467_b200 import Context
cfg = synth.CONFIGS["C2"]
seq = synth.HostSequence(cfg)
u = seq.initial(); A = seq.matrix(1, u)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
ctx = Context(cfg.n, t(A.row_ptr), t(A.col_idx), t(A.val), max_m=cfg.m, max_snapshots=cfg.s, max_k=cfg.k)
rng = np.random.default_rng(0)
base = rng.standard_normal(cfg.n)
for i in range(cfg.s):
    ctx.push_snapshot(t(base + 0.1 ** (i % 6) * rng.standard_normal(cfg.n)))
N = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for i in range(3):
    ctx.build_recycle(cfg.k)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(N):
    ctx.build_recycle(cfg.k)
torch.cuda.synchronize()
print("host ms/call", (time.perf_counter() - t0) / N * 1e3)
