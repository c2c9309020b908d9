"""Device kernel timeline of bench steps (rg_kernel_trace; RG_FLAG_PROFILE): where a system's time goes
between the library's kernels.  Runs `warmup` systems, then traces `n` systems of the bench sequence.
python tools/trace.py C4 [variant] [n] [--no-persist]   -> per-transition gap table + kernel busy share
"Gap" = next kernel's block-0 start minus the previous kernel's last-CTA end on the main chain (launch
latency + ramp + drain; negative when they overlap, e.g. with programmatic dependent launch)."""
import collections
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import synth
from paper_1807_09467_b200 import rg

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "C4"
variant = args[1] if len(args) > 1 else "deflate"
n = int(args[2]) if len(args) > 2 else 2
flags = rg.RG_FLAG_NO_PERSIST if "--no-persist" in sys.argv else 0
cfg = synth.CONFIGS[name]
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
with torch.cuda.stream(st):
    run = bench.GpuRun(cfg, variant, cfg.k, dev, st, profile=True, sell=cfg.fmt == "sell", flags=flags)
    for _ in range(4):
        run.step()
    torch.cuda.synchronize()
    run.ctx.reset_kernel_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n):
        run.step()
    e1.record(st)
    torch.cuda.synchronize()
    ev, total = run.ctx.kernel_trace()
wall_ms = e0.elapsed_time(e1) / n
ev.sort(key=lambda e: e[0])
# pair start/end per kernel name (FIFO)
open_ = collections.defaultdict(list)
iv = []
for t, kind, nm in ev:
    if kind == 0:
        open_[nm].append(t)
    elif kind == 1 and open_[nm]:
        iv.append((open_[nm].pop(0), t, nm))
iv.sort()
side = {"dcgs_ls"}
main = [x for x in iv if x[2] not in side]
busy = collections.Counter()
for s0, s1, nm in iv:
    busy[nm] += s1 - s0
span = (max(x[1] for x in iv) - min(x[0] for x in iv)) if iv else 0
gaps = collections.defaultdict(list)
for a, b in zip(main, main[1:]):
    gaps[(a[2], b[2])].append(b[0] - a[1])
noops = collections.Counter(nm for t, k, nm in ev if k == 2)
print(f"{name} {variant}: {n} systems, {wall_ms:.3f} ms/system (events), {total} trace events, "
      f"traced span {span / 1e6 / n:.3f} ms/system")
print(f"main-chain kernels busy {sum(v for k, v in busy.items() if k not in side) / 1e6 / n:.3f} ms/system; "
      f"sum of gaps {sum(sum(g) for g in gaps.values()) / 1e6 / n:.3f} ms/system")
print("kernel busy (ms/system):", ", ".join(f"{k} {v / 1e6 / n:.3f}" for k, v in busy.most_common(12)))
print("no-op launches per system:", ", ".join(f"{k} {v / n:.1f}" for k, v in noops.most_common(8)))
print(f"{'transition':44s} {'count/sys':>9s} {'mean gap us':>11s} {'total ms/sys':>12s}")
for (a, b), g in sorted(gaps.items(), key=lambda kv: -sum(kv[1])):
    print(f"{a + ' -> ' + b:44s} {len(g) / n:9.1f} {sum(g) / len(g) / 1e3:11.2f} {sum(g) / 1e6 / n:12.3f}")
