"""Short sequence run for profiling: python tools/prof_seq.py CONFIG VARIANT SYSTEMS [sell] [--stats]
With --stats, the per-system kernel statistics (device time, algorithmic bytes) are printed as JSON."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
args = [a for a in sys.argv[1:] if not a.startswith("--")]
stats = "--stats" in sys.argv
cfg = synth.CONFIGS[args[0] if len(args) > 0 else "C2"]
variant = args[1] if len(args) > 1 else "deflate"
T = int(args[2]) if len(args) > 2 else 3
sell = bool(int(args[3])) if len(args) > 3 else cfg.fmt == "sell"
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
with torch.cuda.stream(st):
    run = bench.GpuRun(cfg, variant, cfg.k, dev, st, profile=stats, sell=sell)
    for t in range(T):
        if stats:
            run.ctx.reset_kernel_stats()
        rep = run.step()
        torch.cuda.synchronize()
        if stats:
            ks = {k: v for k, v in run.ctx.kernel_stats().items() if v["launches"] and not k.startswith("p_")}
            print(json.dumps({"system": t + 1, "iterations": rep["iterations"], "kernels": ks}))
print("iters", run.iters)
