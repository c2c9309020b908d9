#!/usr/bin/env python
"""Benchmark of the recycled GMRES(m) hot path on B200 (one JSON line on rank 0).

A STEP is one system of the sequence (every row of SURVEY.md §8a): the next A_t, b_t are generated
in HBM from x_{t-1} (a1), the values are handed to the library (rg_update_matrix), the recycle
space is rebuilt from the snapshot window (a3; C = A W and its QR are rebuilt inside the solve, a4),
the system is solved with the recycled variant (a5-a10), and x_t is pushed as a snapshot (a2).

Default workload: BASELINE.json configs[4] (C5, n = 2,097,152, BSR-64 with 7.31 GB of values,
GMRES(30), k = 20 from 40 snapshots), variant deflate: the largest single-GPU configuration.  When
--warmup + --steps exceeds the config's sequence length (C5: 20 systems) the sequence continues with
the same generator (C5: A_t = A_{t-1} o (1 + 0.01 xi_t), b fixed).  Other configs: --config C1..C4,
--variant plain|augment|deflate|oblique|orthogonal.

  value      seconds per system (device time, CUDA events on the library's stream), whole job:
             max-over-ranks time / (systems solved by all ranks)
  e2e        the same metric through the public API with HOST buffers (host generator, H2D of
             A_t values / b_t / snapshot, D2H of x_t inside the timed region)
  roofline   the dominant kernel's algorithmic bytes / its measured device time (%globaltimer
             stamps inside the kernels: launches live inside CUDA graphs, where host-side events
             cannot bracket single kernels), against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the oracle (plain C, deterministic OpenMP threads on all online cores) on the first
             timed systems of the same workload, bounded to ~--cpu-budget seconds
  phases_ms_per_step  device time per system of the recycle build (a3), the generation of A_t, b_t (the
             synthetic source, not a library kernel), the solve (a4-a10) and the snapshot push (a2),
             from events at the phase boundaries of every timed step; `value` has all four

--impl reference runs the oracle (the reference arm for this tier) on the same config.
Multi-GPU (torchrun): independent replicas, one sequence per rank, no collective on the data
path ("replicas only"); barrier + max-over-ranks timing.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "recycled GMRES(m) sec per system & sequence; SpMV/Arnoldi HBM GB/s vs peak"
UNIT = "s/system"


# ---------------------------------------------------------------------------------------- helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def reduce_max(value: float, dist_on: bool, device=None) -> float:
    """Max over ranks (the contract's timing rule)."""
    if not dist_on:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed_replicas(step, steps, warmup, dist_on, device=None, timer="cuda", between=None, stream=None):
    """The contract's timing skeleton, shared by every rank: `warmup` untimed steps, barrier,
    exactly `steps` timed steps (per-step device events on `stream`, or host clock for
    timer="cpu"), barrier, max over ranks.  `between` runs before each timed step, outside the
    timed window (the L2 flush).  Returns (per_step_seconds, local_total, max_total)."""
    for _ in range(warmup):
        step()
    if timer == "cuda":
        import torch
        torch.cuda.synchronize()
    if dist_on:
        import torch.distributed as dist
        dist.barrier()
    per = []
    if timer == "cuda":
        import torch
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        for i in range(steps):
            if between:
                between()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        per = [a.elapsed_time(b) / 1e3 for a, b in evs]
    else:
        for i in range(steps):
            if between:
                between()
            t0 = time.perf_counter()
            step()
            per.append(time.perf_counter() - t0)
    if dist_on:
        import torch.distributed as dist
        dist.barrier()
    t_local = sum(per)
    return per, t_local, reduce_max(t_local, dist_on, device)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region: NVML polled
    every 2 ms from a background thread (nvidia-smi's 100 ms loop would see one sample of a
    ~0.1 s region); falls back to `nvidia-smi -lms 100` when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.thread = None
        self.samples = []
        self.path = os.path.join("/tmp", f"rg_clocks_{os.getpid()}.csv")

    def _poll(self, pynvml, h):
        bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self.stop:
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(mx), {n for n, b in bits.items() if rs & b}))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        self.stop = False
        try:
            import threading

            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.thread = threading.Thread(target=self._poll, args=(pynvml, h), daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.stop = True
        if self.thread is not None:
            self.thread.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.thread is not None:
            if not self.samples:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no NVML samples"], "samples": 0}
            reasons = set().union(*[r for _, _, r in self.samples])
            return {"sm_mhz": statistics.median([s for s, _, _ in self.samples]),
                    "sm_max_mhz": max(m for _, m, _ in self.samples), "reasons": sorted(reasons),
                    "samples": len(self.samples), "source": "nvml, 2 ms"}
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, p[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi, 100 ms"}


# ---------------------------------------------------------------------------------------- our arm
class GpuRun:
    """One replica: the library context plus the device-side sequence generator."""

    def __init__(self, cfg, variant, k, device, stream, profile, sell, precond=None, sync_build=False, flags=0,
                 warm=False):
        import torch

        import synth
        from paper_1807_09467_b200 import Context, rg
        self.torch, self.cfg, self.variant, self.k = torch, cfg, variant, k
        self.sync_build = sync_build   # True: rg_build_recycle returns k_eff, sigma (host sync)
        self.warm = warm               # True: x0 = x_{t-1} (SURVEY A4's warm-started reference row)
        self.dev = device
        self.stream = stream
        self.gen = synth.DeviceSequence(cfg, device)
        u0 = torch.from_numpy(self.gen.host.initial()).to(device)
        self.x = torch.zeros(cfg.n, dtype=torch.float64, device=device)
        self.x.copy_(u0)
        self.gen.fill(1, self.x)
        flags = flags | (rg.RG_FLAG_PROFILE if profile else 0)
        self.ctx = Context(cfg.n, self.gen.row_ptr, self.gen.col_idx, self.gen.val,
                           fmt="bsr" if cfg.kind == "bsr" else "csr", block=cfg.B if cfg.kind == "bsr" else 1,
                           sell_C=32 if sell else 0, max_m=cfg.m, max_snapshots=cfg.s,
                           max_k=max(k, 1), stream=stream.cuda_stream, flags=flags)
        if precond:
            self.ctx.set_preconditioner("ssor", precond)   # library greedy multicolour order
        self.t = 0
        self.iters = []
        self.nsnap = 0
        self.vals_ptr, _ = self.ctx.values_ptr()
        self.nnz = int(self.gen.col_idx.numel())
        self.phase_ev = None           # a list: step() appends its 5 phase-boundary events (run_ours)

    def _mark(self, evs):
        if evs is not None:
            e = self.torch.cuda.Event(enable_timing=True)
            e.record(self.stream)
            evs.append(e)

    def step(self, x_prev=None, push=None, history_cap=0):
        """One system t of the sequence, entirely on the device (inputs resident in HBM).
        Teacher forcing (tests): x_prev (device) replaces x_{t-1} before A_t, b_t are generated, and
        push (device) is the snapshot pushed instead of the solver's x_t."""
        cfg = self.cfg
        self.t += 1
        if x_prev is not None:
            self.x.copy_(x_prev)
        evs = [] if self.phase_ev is not None else None
        self._mark(evs)
        # a3 first: W depends only on the snapshot window, not on A_t, so the asynchronous build is issued
        # before the generator and its completion (which the solve waits for on the host) overlaps the
        # generation of A_t instead of leaving a bubble before the solve (tools/trace.py: ~0.1 ms/system)
        if self.variant != "plain" and self.nsnap > 0:
            if self.sync_build:
                self.k_eff, self.sigma = self.ctx.build_recycle(self.k)
            else:                                      # a3, asynchronous (a4 happens inside the solve)
                self.ctx.build_recycle(self.k, deferred=True)
        self._mark(evs)
        if cfg.kind == "9pt":                          # C3: A is the same for the whole sequence
            self.gen.fill(self.t, self.x)              # (b_t only)
        else:                                          # A_t, b_t from x_{t-1}, written straight into
            self.gen.fill(self.t, self.x, val_ptr=self.vals_ptr)   # the solver's value buffer (a1)
            self.ctx.update_values_inplace(self.nnz)
        self._mark(evs)
        rep = self.ctx.solve(self.gen.b, self.x, x0=self.x if self.warm else None, m=cfg.m, variant=self.variant,
                             tol=cfg.tol, history_cap=history_cap)
        if not rep["converged"]:
            raise RuntimeError(f"system {self.t} did not converge: {rep}")
        self._mark(evs)
        self.ctx.push_snapshot(self.x if push is None else push)   # a2
        self._mark(evs)
        if evs is not None:
            self.phase_ev.append(evs)
        self.nsnap += 1
        self.iters.append(rep["iterations"])
        return rep


class HostE2ERun:
    """The same sequence through the public API with HOST buffers (pinned), host generator."""

    def __init__(self, cfg, variant, k, device, stream, sell, precond=None):
        import torch

        import synth
        from paper_1807_09467_b200 import Context
        self.torch, self.cfg, self.variant, self.k = torch, cfg, variant, k
        self.seq = synth.HostSequence(cfg)
        u0 = self.seq.initial()
        A1 = self.seq.matrix(1, u0)
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        self.x = torch.zeros(cfg.n, dtype=torch.float64).pin_memory()
        self.x.copy_(torch.from_numpy(u0))
        self.val = pin(A1.val)
        self.b = torch.zeros(cfg.n, dtype=torch.float64).pin_memory()
        self.ctx = Context(cfg.n, pin(A1.row_ptr), pin(A1.col_idx), self.val,
                           fmt="bsr" if cfg.kind == "bsr" else "csr", block=cfg.B if cfg.kind == "bsr" else 1,
                           sell_C=32 if sell else 0, max_m=cfg.m, max_snapshots=cfg.s,
                           max_k=max(k, 1), stream=stream.cuda_stream)
        if precond:
            self.ctx.set_preconditioner("ssor", precond)
        self.t = 0
        self.nsnap = 0
        self.h2d = 0
        self.d2h = 0

    def prepare(self):
        """Host-side input generation for the next system (the synthetic data source, not the API):
        A_t values and b_t into the pinned buffers."""
        self.t += 1
        xn = self.x.numpy()
        hm = self.seq.matrix(self.t, xn)
        self.val.numpy()[:] = hm.val
        self.b.numpy()[:] = self.seq.rhs(self.t, xn)

    def step(self):
        """The public-API calls of one system with HOST buffers: H2D of A_t values and b_t, recycle
        build, solve (x_t D2H into host memory), snapshot push (H2D)."""
        cfg = self.cfg
        self.ctx.update_matrix(self.val)
        if self.variant != "plain" and self.nsnap > 0:
            self.ctx.build_recycle(self.k, deferred=True)
        rep = self.ctx.solve(self.b, self.x, m=cfg.m, variant=self.variant, tol=cfg.tol)
        self.ctx.push_snapshot(self.x)
        self.nsnap += 1
        self.h2d = 8 * (self.val.numel() + 2 * cfg.n)   # values, b, snapshot
        self.d2h = 8 * cfg.n                            # x_t
        return rep


def flush_l2(buf):
    buf.add_(1.0)   # 256 MiB write > 126 MB L2


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_time(cfg, variant, k, systems, budget_s=30.0, precond=None, first=1):
    """The oracle (plain C fp64, deterministic OpenMP threads on all online cores) on its own
    sequence: systems 1..first-1 are solved untimed (they fill the snapshot window), then systems
    first..systems are timed until `budget_s` is spent (at least one).  precond = omega: right SSOR
    in the greedy multicolour order of tests/coloring.py.  Returns (times, iterations, threads)."""
    import oracle
    import synth
    oracle.set_threads(os.cpu_count() or 1)
    seq = synth.HostSequence(cfg)
    u = seq.initial()
    pc = None
    if precond:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from coloring import greedy_colors
        A1 = seq.matrix(1, u)
        pc = (oracle.ssor_order(greedy_colors(A1.n, A1.row_ptr, A1.col_idx)), precond)
    X = []
    times = []
    its = []
    for t in range(1, systems + 1):
        A = oracle.Matrix.from_host(seq.matrix(t, u))
        b = seq.rhs(t, u)
        t0 = time.perf_counter()
        W = None
        if variant != "plain" and X:
            W, _, _ = oracle.recycle_basis(np.stack(X[-cfg.s:], 1), k)
        r = oracle.solve(A, b, m=cfg.m, variant=variant, W=W, tol=cfg.tol, precond=pc)
        if t >= first:
            times.append(time.perf_counter() - t0)
            its.append(r["iterations"])
        u = r["x"]
        X.append(u)
        if times and sum(times) > budget_s:
            break
    return times, its, oracle.threads()


def run_ours(args, cfg):
    import torch
    ws, rank, local = dist_env()
    dist_on = ws > 1
    if dist_on:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    stream = torch.cuda.Stream(device)
    k = args.k or cfg.k
    flush = torch.zeros(32 * 1024 * 1024, dtype=torch.float64, device=device)
    with torch.cuda.stream(stream):
        sell = (cfg.fmt == "sell") if args.sell < 0 else bool(args.sell)
        from paper_1807_09467_b200 import rg as _rg
        run = GpuRun(cfg, args.variant, k, device, stream, profile=not args.no_profile, sell=sell,
                     precond=args.omega if args.precond == "ssor" else None,
                     flags=(_rg.RG_FLAG_NO_GRAPH if args.no_graph else 0) |
                           (_rg.RG_FLAG_NO_PERSIST if args.no_persist else 0))
        for _ in range(args.warmup):
            run.step()
        torch.cuda.synchronize()
        run.ctx.reset_kernel_stats()
        gen0 = run.gen.launches
        run.phase_ev = []
        with ClockSampler(local) as clk:
            per, t_local, t_max = timed_replicas(run.step, args.steps, 0, dist_on, device, "cuda",
                                                 between=lambda: flush_l2(flush), stream=stream)
        kstats = run.ctx.kernel_stats()
        gen_launches = run.gen.launches - gen0
        # per-system setup / generation / solve times, from events on the library's stream at
        # the phase boundaries of every timed step (the solve includes a4, C = A W, which needs A_t)
        names = ["recycle_build_a3", "generation_and_a1", "solve_a4_to_a10", "snapshot_push_a2"]
        phases = {nm: sum(ev[i].elapsed_time(ev[i + 1]) for ev in run.phase_ev) / len(run.phase_ev)
                  for i, nm in enumerate(names)}
        run.phase_ev = None
        value = t_max / (args.steps * ws)
        timed_iters = run.iters[args.warmup:]

        # e2e through the public API with host buffers
        e2e = None
        if not args.no_e2e:
            hrun = HostE2ERun(cfg, args.variant, k, device, stream, sell,
                              precond=args.omega if args.precond == "ssor" else None)
            for _ in range(min(args.warmup, 2)):
                hrun.prepare()
                hrun.step()
            torch.cuda.synchronize()
            if dist_on:
                torch.distributed.barrier()
            ke = max(1, min(args.steps, args.e2e_steps))
            te_local = 0.0
            for _ in range(ke):
                hrun.prepare()                 # host generation of the inputs: outside the clock
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                hrun.step()                    # API calls incl. H2D inputs and D2H of x_t
                torch.cuda.synchronize()
                te_local += time.perf_counter() - t0
            te = reduce_max(te_local, dist_on, device)
            e2e = {"value": te / (ke * ws), "unit": UNIT, "h2d_bytes_per_step": hrun.h2d,
                   "d2h_bytes_per_step": hrun.d2h, "steps": ke,
                   "scope": "public API calls with pinned HOST buffers per system: rg_update_matrix (H2D values), "
                            "rg_build_recycle, rg_solve (H2D b, D2H x), rg_push_snapshot (H2D x); the host "
                            "generation of A_t, b_t (synthetic data source) is outside the clock"}

        # the recycled sequence against plain GMRES(m) on the GPU (north_star: "the recycled solver's
        # end-to-end sequence time reported against plain GMRES(m)"): the same config as a plain
        # sequence, same warm-up, same timed systems, same device timing and L2 flushes
        vs_plain = None
        if not args.no_vs_plain and args.variant != "plain":
            hrun = None
            run.ctx.close()
            prun = GpuRun(cfg, "plain", k, device, stream, profile=False, sell=sell,
                          precond=args.omega if args.precond == "ssor" else None)
            for _ in range(args.warmup):
                prun.step()
            torch.cuda.synchronize()
            pper, _, pt_max = timed_replicas(prun.step, args.steps, 0, dist_on, device, "cuda",
                                             between=lambda: flush_l2(flush), stream=stream)
            pits = prun.iters[args.warmup:]
            prun.ctx.close()
            # warm-started plain GMRES(m): x0 = x_{t-1} (the paper compares initial guesses,
            # PAPER.md:405-436, Table 2)
            wrun = GpuRun(cfg, "plain", k, device, stream, profile=False, sell=sell,
                          precond=args.omega if args.precond == "ssor" else None, warm=True)
            for _ in range(args.warmup):
                wrun.step()
            torch.cuda.synchronize()
            _, _, wt_max = timed_replicas(wrun.step, args.steps, 0, dist_on, device, "cuda",
                                          between=lambda: flush_l2(flush), stream=stream)
            wits = wrun.iters[args.warmup:]
            wrun.ctx.close()
            vs_plain = {"variant": "plain", "value": pt_max / (args.steps * ws), "unit": UNIT,
                        "sequence_s": pt_max, "iterations_timed": pits,
                        "iterations_total": sum(pits), "recycled_iterations_total": sum(timed_iters),
                        "recycled_sequence_s": t_max,
                        "sequence_speedup": round(pt_max / t_max, 4),
                        "warm_plain": {"value": wt_max / (args.steps * ws), "unit": UNIT, "sequence_s": wt_max,
                                       "iterations_total": sum(wits), "sequence_speedup": round(wt_max / t_max, 4),
                                       "scope": "plain GMRES(m) with x0 = x_{t-1} (SURVEY A4), same systems"},
                        "scope": "the same systems t of a free-running plain GMRES(m) sequence (its own "
                                 "x_{t-1} drives A_t, b_t), timed like the main line"}

    if rank != 0:
        if dist_on:
            torch.distributed.destroy_process_group()
        return
    # roofline of the dominant kernel (largest summed device time in the timed region)
    peak, peak_kind = measured_peaks()
    work = {kname: s for kname, s in kstats.items()
            if s["launches"] > 0 and s["ms"] > 0 and not kname.startswith("p_")}
    dom = max(work, key=lambda kname: work[kname]["ms"]) if work else None
    roof = None
    if dom:
        s = work[dom]
        bytes_per = s["bytes"] / s["launches"]
        ms_per = s["ms"] / s["launches"]
        achieved = bytes_per / (ms_per * 1e-3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", f"traffic_{cfg.name}_{args.variant}.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get(dom)
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": bytes_per, "avg_launch_us": ms_per * 1e3,
                "share_of_step": round(s["ms"] / 1e3 / t_local, 4)}
        if roof["frac"] > 1.0:
            # MEASURED_PEAKS.json's hbm_gbs is a COPY (read + write) rate; a read-dominated stream runs a
            # few percent above it (flat 16-byte read probe on the B200: 6.96 TB/s, profiles/r02/)
            ratio = f" (DRAM traffic {traffic / bytes_per:.3f}x algorithmic)" if traffic else ""
            roof["note"] = ("peak is the measured read+write copy rate; this kernel is a read-dominated stream"
                            + ratio + ", which exceeds a copy by a few percent")
    # kernel launches in the timed region: device-counted executions (incl. launches that found nothing
    # to do), the library's host-launched kernels, and the input generator's kernels.  Not summed:
    # the p_* phase timers inside the persistent solve and "ssor" (per application; its kernels are
    # counted in "ssor_sweep_kernels").  Under profiling, a "gram" entry counts its two kernels as one
    # (the second is in "host_launched").
    launches = sum(s["launches"] + s["noop"] for kname, s in kstats.items()
                   if not kname.startswith("p_") and kname != "ssor") + gen_launches
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        first = args.warmup + 1                      # the first timed system of this run
        times, its, nth = oracle_time(cfg, args.variant, k, args.warmup + args.steps, budget_s=args.cpu_budget,
                                      precond=args.omega if args.precond == "ssor" else None, first=first)
        cpu = {"value": sum(times) / len(times), "unit": UNIT, "cores": nth, "kind": "oracle",
               "cpu_model": cpu_model(), "online_cores": os.cpu_count(),
               "sample": f"{cfg.name} systems {first}..{first + len(times) - 1} of the oracle's own sequence "
                         f"({args.variant}, iterations {its}; the timed region's first systems, bounded to "
                         f"~{args.cpu_budget:.0f} s; systems 1..{first - 1} solved untimed to fill the window), "
                         f"plain C fp64, deterministic OpenMP threads"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators, synth/)",
        "config": {"workload": f"{cfg.name}: BASELINE.json configs[{cfg.cid - 1}]", "variant": args.variant,
                   "precond": f"right SSOR(omega={args.omega}), multicolour" if args.precond == "ssor" else "none",
                   "n": cfg.n, "m": cfg.m, "k": k, "s": cfg.s, "fmt": cfg.fmt,
                   "device_format": "SELL-32" if sell else ("BSR-64" if cfg.kind == "bsr" else "CSR"),
                   "tol": cfg.tol,
                   "systems_timed": f"t={args.warmup + 1}..{args.warmup + args.steps}" + (
                       f" (the config's sequence has {cfg.systems}; continued by the same generator)"
                       if args.warmup + args.steps > cfg.systems else ""),
                   "iterations_timed": timed_iters,
                   "l2": "flushed (256 MiB write) between steps, outside the timed events",
                   "parallelism": f"replicas x{ws}"},
        "per_step_s": [round(p, 6) for p in per],
        "sequence_s": t_max,
        "phases_ms_per_step": {**{nm: round(v, 4) for nm, v in phases.items()},
                               "scope": "rank 0, device events on the library's stream at the phase boundaries "
                                        "of each timed step; generation = the synthetic source writing A_t, b_t "
                                        "(in place into the library's value buffer), not a library kernel; "
                                        "`value` includes all four"},
        "vs_plain": vs_plain,
        "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "gpu_launches": launches,
        "clocks": clk.summary(),
        "kernels": {kname: {"launches": s["launches"], "noop": s["noop"], "ms": round(s["ms"], 4),
                            "tail_ms": round(s["tail_ms"], 4),
                            "GBps": round(s["bytes"] / (s["ms"] * 1e-3) / 1e9, 1) if s["ms"] > 0 else None}
                    for kname, s in kstats.items() if s["launches"] + s["noop"] > 0},
    }
    print(json.dumps(line))
    if dist_on:
        torch.distributed.destroy_process_group()


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    k = args.k or cfg.k
    n_sys = args.warmup + args.steps
    timed, its, nth = oracle_time(cfg, args.variant, k, n_sys, budget_s=1e9,
                                  precond=args.omega if args.precond == "ssor" else None, first=args.warmup + 1)
    v = sum(timed) / len(timed)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators, synth/)",
            "config": {"workload": f"{cfg.name}: BASELINE.json configs[{cfg.cid - 1}]", "variant": args.variant,
                       "n": cfg.n, "m": cfg.m, "k": k, "s": cfg.s, "iterations": its,
                       "systems_timed": f"t={args.warmup + 1}..{n_sys}" + (
                           f" (the config's sequence has {cfg.systems}; continued by the same generator)"
                           if n_sys > cfg.systems else "")},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nth, "kind": "oracle", "cpu_model": cpu_model(),
                             "online_cores": os.cpu_count(),
                             "sample": f"{cfg.name} systems {args.warmup + 1}..{n_sys} of the oracle's own sequence "
                                       f"(1..{args.warmup} untimed), deterministic OpenMP threads"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed systems; default: the rest of the config's sequence after the warm-up "
                         "(C2: 47 of 50) for our arm, 3 for --impl reference")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--variant", default="deflate", choices=["plain", "augment", "deflate", "oblique", "orthogonal"])
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--precond", default="none", choices=["none", "ssor"],
                    help="right SSOR preconditioner in a multicolour order (SURVEY NEXT #2)")
    ap.add_argument("--omega", type=float, default=1.0)
    ap.add_argument("--sell", type=int, default=-1, help="1: pack CSR to SELL-32 inside the library, "
                    "0: keep CSR, -1: config default")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-persist", action="store_true",
                    help="RG_FLAG_NO_PERSIST: the CUDA-graph path even where the persistent kernel would run")
    ap.add_argument("--no-graph", action="store_true",
                    help="RG_FLAG_NO_GRAPH: launch the solve's kernels one by one (ncu cannot profile kernels "
                         "inside conditional CUDA graphs); for profiler captures, not for timing")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-vs-plain", action="store_true",
                    help="skip the plain GMRES(m) sequence timed beside the recycled one")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: the contract asks for >= 3 warm-up steps", file=sys.stderr)
    import synth
    cfg = synth.CONFIGS[args.config]
    if args.steps is None:
        args.steps = max(1, cfg.systems - args.warmup)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
