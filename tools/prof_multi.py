"""Run short sequences of several configs in ONE process (for one ncu invocation covering them):
python tools/prof_multi.py C3:deflate:3 C4:deflate:3 C5:deflate:2
Each entry = CONFIG:VARIANT:SYSTEMS.  Use with RG_NO_GRAPH=1 RG_NO_PERSIST=1 so that ncu sees the
individual kernels (it cannot profile kernels inside conditional graph nodes)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
for spec in sys.argv[1:]:
    name, variant, T = spec.split(":")
    cfg = synth.CONFIGS[name]
    with torch.cuda.stream(st):
        run = bench.GpuRun(cfg, variant, cfg.k, dev, st, profile=False, sell=cfg.fmt == "sell")
        for _ in range(int(T)):
            run.step()
        torch.cuda.synchronize()
    print(name, variant, "iters", run.iters, flush=True)
    del run
    torch.cuda.empty_cache()
