"""Where does a bench step's device time go?  CUDA events between the API calls of bench.GpuRun.step
(same calls, same stream), averaged over N systems after warm-up:  python tools/step_gaps.py C2 20"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
names = ["fill", "update", "build_recycle", "solve", "push"]
acc = [0.0] * len(names)
with torch.cuda.stream(st):
    run = bench.GpuRun(cfg, "deflate", cfg.k, dev, st, profile=False, sell=cfg.fmt == "sell")
    for _ in range(3):
        run.step()
    for it in range(N):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
        run.t += 1
        ev[0].record(st)
        if cfg.kind == "9pt":
            run.gen.fill(run.t, run.x)
        else:
            run.gen.fill(run.t, run.x, val_ptr=run.vals_ptr)
        ev[1].record(st)
        if cfg.kind != "9pt":
            run.ctx.update_values_inplace(run.nnz)
        ev[2].record(st)
        import time as _t
        h0 = _t.perf_counter()
        run.ctx.build_recycle(run.k)
        hb = _t.perf_counter() - h0
        host_br = globals().setdefault("host_br", [])
        host_br.append(hb)
        ev[3].record(st)
        rep = run.ctx.solve(run.gen.b, run.x, m=cfg.m, variant="deflate", tol=cfg.tol)
        ev[4].record(st)
        run.ctx.push_snapshot(run.x)
        ev[5].record(st)
        torch.cuda.synchronize()
        for i in range(len(names)):
            acc[i] += ev[i].elapsed_time(ev[i + 1])
        acc_solve_dev = rep["ms_total"]
tot = sum(acc)
print({n: round(a / N, 4) for n, a in zip(names, acc)}, "total ms/system", round(tot / N, 4),
      "host ms in build_recycle", round(1e3 * sum(host_br) / len(host_br), 4))
