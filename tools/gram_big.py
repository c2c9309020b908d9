"""Gram / X*M at C4 window sizes (n = 2M, s = 32) through rg_build_recycle, for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1807_09467_b200 import Context
cfg = synth.CONFIGS["C4"]
n = cfg.n
rp = torch.arange(n + 1, dtype=torch.int32, device="cuda")
ci = torch.arange(n, dtype=torch.int32, device="cuda")
v = torch.ones(n, dtype=torch.float64, device="cuda")
ctx = Context(n, rp, ci, v, max_m=8, max_snapshots=32, max_k=16)
g = torch.Generator(device="cuda").manual_seed(0)
for i in range(32):
    ctx.push_snapshot(torch.randn(n, dtype=torch.float64, device="cuda", generator=g))
for i in range(3):
    ctx.build_recycle(16)
torch.cuda.synchronize()
print("ok")
