"""Persistent-kernel vs graph-path crossover: ms/system of the same seeded sequence through both paths
(RG_FLAG_NO_PERSIST), for a config resized to N (grid side) and a variant.
python tools/crossover.py C3 768 deflate [ssor]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import synth
from paper_1807_09467_b200 import rg

name, N, variant = sys.argv[1], int(sys.argv[2]), sys.argv[3]
pre = 1.0 if len(sys.argv) > 4 and sys.argv[4] == "ssor" else None
cfg = synth.CONFIGS[name].reduced(N)
dev = torch.device("cuda", 0)
out = []
for rep in range(2):
    for flags in (0, rg.RG_FLAG_NO_PERSIST):
        st = torch.cuda.Stream(dev)
        with torch.cuda.stream(st):
            run = bench.GpuRun(cfg, variant, cfg.k, dev, st, profile=True, sell=cfg.fmt == "sell", precond=pre, flags=flags)
            for _ in range(3):
                run.step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(6):
                run.step()
            e1.record(st)
            torch.cuda.synchronize()
            ks = run.ctx.kernel_stats()
            path = "persistent" if ks["persistent_solve"]["launches"] else "graph"
            print(f"{name} N={N} n={cfg.n} {variant}{' ssor' if pre else ''} flags={flags} path={path}: "
                  f"{e0.elapsed_time(e1) / 6:.4f} ms/system, iterations {sum(run.iters[-6:])}", flush=True)
            run.ctx.close()
