"""Short sequence run for profiling: python tools/prof_seq.py CONFIG VARIANT SYSTEMS [sell]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
variant = sys.argv[2] if len(sys.argv) > 2 else "deflate"
T = int(sys.argv[3]) if len(sys.argv) > 3 else 3
sell = bool(int(sys.argv[4])) if len(sys.argv) > 4 else cfg.fmt == "sell"
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
with torch.cuda.stream(st):
    run = bench.GpuRun(cfg, variant, cfg.k, dev, st, profile=False, sell=sell)
    for _ in range(T):
        rep = run.step()
    torch.cuda.synchronize()
print("iters", run.iters)
