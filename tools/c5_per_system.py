"""Per-system device times of the C5 bench step's kernels as the recycle dimension grows
(python tools/c5_per_system.py [systems]): where the step's growth with k_eff goes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth

def main():
    nsys = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    cfg = synth.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "C5"]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        run = bench.GpuRun(cfg, "deflate", cfg.k, dev, stream, profile=True, sell=(cfg.fmt == "sell"))
        names = ["spmv_step", "spmv_plain", "spmv_res", "cbuild", "gram", "jacobi", "orth_dots1", "orth_upd_dots2",
                 "orth_upd_norm_ls", "dcgs_dots_ls", "dcgs_update"]
        print("t iters " + " ".join(names))
        for t in range(1, nsys + 1):
            run.ctx.reset_kernel_stats()
            rep = run.step()
            torch.cuda.synchronize()
            ks = run.ctx.kernel_stats()
            print(t, rep["iterations"], " ".join(f"{ks[n]['ms']:.3f}" if n in ks else "-" for n in names), flush=True)

if __name__ == "__main__":
    main()
