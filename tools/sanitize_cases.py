"""Small solves on every execution path, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): tools/sanitize.sh runs this under each tool.  Exits non-zero if a solve fails.
  persistent   C1 (one 1024-thread CTA) and C4 at N = 20 (n = 8,000: several CTAs, grid barriers,
               neighbour sync, flag-carrying reductions), plain / augment / deflate / oblique
  graph        RG_FLAG_NO_PERSIST: DCGS2 kernels (k_dk1 / k_dk2 or their TMA-streamed variants)
  cgs2         RG_FLAG_CGS2 | RG_FLAG_NO_PERSIST: classical CGS2 kernels
  ssor         right multicolour SSOR (persistent and graph)
  bsr          C5 at E = 3 (BSR-64: TMA SpMV, tensor-map TMA + DMMA SpMM, fused start residual)
python tools/sanitize_cases.py [case ...]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1807_09467_b200 import Context, rg  # noqa: E402


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def sequence(cfg, variants, flags=0, systems=3, precond=None, x0=False):
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    A1 = seq.matrix(1, u)
    ctx = Context(cfg.n, t(A1.row_ptr), t(A1.col_idx), t(A1.val), fmt=A1.fmt, block=A1.block,
                  max_m=cfg.m, max_snapshots=cfg.s, max_k=cfg.k, flags=flags)
    if precond:
        ctx.set_preconditioner("ssor", precond)
    x = torch.zeros(cfg.n, dtype=torch.float64, device="cuda")
    for step in range(1, systems + 1):
        A = seq.matrix(step, u)
        ctx.update_matrix(t(A.val))
        b = t(seq.rhs(step, u))
        for v in variants:
            if step > 1 and v != "plain":
                ctx.build_recycle(cfg.k)
            rep = ctx.solve(b, x, x0=t(u) if x0 else None, m=cfg.m, variant=v, tol=cfg.tol)
            if not rep["converged"]:
                raise SystemExit(f"{cfg.name} {v} flags={flags}: not converged {rep}")
        u = x.cpu().numpy().copy()
        ctx.push_snapshot(x)
    ctx.close()


def main(cases):
    C1 = synth.CONFIGS["C1"]
    C4s = synth.CONFIGS["C4"].reduced(20, k=4, s=8)
    C5s = synth.CONFIGS["C5"].reduced(3, k=3, s=6)
    run = {
        "persistent": lambda: (sequence(C1, ["plain", "augment", "deflate", "oblique"]),
                               sequence(C4s, ["plain", "augment", "deflate"])),
        "graph": lambda: sequence(C4s, ["plain", "augment", "deflate", "oblique"], flags=rg.RG_FLAG_NO_PERSIST),
        "cgs2": lambda: sequence(C4s, ["deflate", "augment"], flags=rg.RG_FLAG_NO_PERSIST | rg.RG_FLAG_CGS2),
        "ssor": lambda: (sequence(C4s, ["deflate"], precond=1.0),
                         sequence(C4s, ["deflate"], flags=rg.RG_FLAG_NO_PERSIST, precond=1.0)),
        "bsr": lambda: (sequence(C5s, ["deflate", "augment"]), sequence(C5s, ["deflate"], x0=True)),
    }
    for c in cases or list(run):
        run[c]()
        print("ok", c, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
