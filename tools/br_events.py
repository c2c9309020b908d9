"""GPU-side duration of rg_build_recycle inside the C2 sequence (events around the call)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
cfg = synth.CONFIGS["C2"]
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
with torch.cuda.stream(st):
    run = bench.GpuRun(cfg, "deflate", cfg.k, dev, st, profile=True, sell=False)
    for _ in range(25):
        run.step()
    torch.cuda.synchronize()
    run.ctx.reset_kernel_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot_gpu = tot_host = 0.0
    for _ in range(20):
        torch.cuda.synchronize()
        e0.record(st)
        t0 = time.perf_counter()
        run.ctx.build_recycle(cfg.k)
        th = time.perf_counter() - t0
        e1.record(st)
        torch.cuda.synchronize()
        tot_gpu += e0.elapsed_time(e1)
        tot_host += th
    print("build_recycle: GPU span ms", tot_gpu / 20, "host ms", tot_host / 20 * 1e3)
    print({k: (v["launches"], round(v["ms"] / 20, 4)) for k, v in run.ctx.kernel_stats().items() if v["launches"]})
