"""Per-step timeline of the bench's API sequence: device time between CUDA events recorded after each
call (on the library's stream) and host time of each call, averaged over N systems after warm-up.
python tools/timeline.py C2 20 [variant]"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 20
variant = sys.argv[3] if len(sys.argv) > 3 else "deflate"
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
names = ["fill", "update", "build", "solve", "push"]
dacc = [0.0] * len(names)
hacc = [0.0] * len(names)
with torch.cuda.stream(st):
    run = bench.GpuRun(cfg, variant, cfg.k, dev, st, profile=True, sell=cfg.fmt == "sell")
    for _ in range(3):
        run.step()
    torch.cuda.synchronize()
    run.ctx.reset_kernel_stats()
    for it in range(N):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
        h = [0.0] * (len(names) + 1)
        run.t += 1
        h[0] = time.perf_counter()
        ev[0].record(st)
        if cfg.kind == "9pt":
            run.gen.fill(run.t, run.x)
        else:
            run.gen.fill(run.t, run.x, val_ptr=run.vals_ptr)
        ev[1].record(st); h[1] = time.perf_counter()
        if cfg.kind != "9pt":
            run.ctx.update_values_inplace(run.nnz)
        ev[2].record(st); h[2] = time.perf_counter()
        if variant != "plain":
            run.ctx.build_recycle(run.k, deferred=True)
        ev[3].record(st); h[3] = time.perf_counter()
        rep = run.ctx.solve(run.gen.b, run.x, m=cfg.m, variant=variant, tol=cfg.tol)
        ev[4].record(st); h[4] = time.perf_counter()
        run.ctx.push_snapshot(run.x)
        ev[5].record(st); h[5] = time.perf_counter()
        torch.cuda.synchronize()
        for i in range(len(names)):
            dacc[i] += ev[i].elapsed_time(ev[i + 1])
            hacc[i] += (h[i + 1] - h[i]) * 1e3
    ks = run.ctx.kernel_stats()
print("device ms/system", {n: round(a / N, 4) for n, a in zip(names, dacc)}, "total", round(sum(dacc) / N, 4))
print("host   ms/system", {n: round(a / N, 4) for n, a in zip(names, hacc)}, "total", round(sum(hacc) / N, 4))
print("kernels us/system", {k: round(v["ms"] * 1e3 / N, 1) for k, v in ks.items() if v["ms"] > 0 and not k.startswith("p_")})
