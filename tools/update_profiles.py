"""Copy a capture directory (tools/gpu_round_capture.sh output) into profiles/: the default bench line,
the per-config lines and table, the ncu launch list + summary, the k_solve_persistent / k_cbuild ncu
--set full summaries (numbers only; the .ncu-rep files stay out of git) and the C2 timelines.
python tools/update_profiles.py gpurun_out/cap3"""
import collections
import csv
import glob
import json
import os
import re
import shutil
import subprocess
import sys

cap = sys.argv[1]
P = "profiles"
os.makedirs(f"{P}/r01_lines", exist_ok=True)
shutil.copy(f"{cap}/bench_default.json", f"{P}/r01_bench_default_C2.json")
open(f"{P}/r01_bench_default_C2.json", "w").write(open(f"{cap}/bench_default.json").read().strip().splitlines()[-1] + "\n")
for f in glob.glob(f"{cap}/bench_*.json"):
    open(f"{P}/r01_lines/{os.path.basename(f)}", "w").write(open(f).read().strip().splitlines()[-1] + "\n")
for f in ("timeline_C2.txt", "timeline_C2_plain.txt"):
    if os.path.exists(f"{cap}/{f}"):
        shutil.copy(f"{cap}/{f}", f"{P}/r01_{f}")

# per-config table
rows = []
for f in sorted(glob.glob(f"{P}/r01_lines/bench_*.json")):
    d = json.loads(open(f).read())
    vp = d.get("vs_plain") or {}
    c = d["config"]
    rows.append((c["workload"][:2], c["variant"], "SSOR" if c["precond"] != "none" else "-", d["value"] * 1e3,
                 sum(c["iterations_timed"]), len(c["iterations_timed"]), vp.get("value", 0) * 1e3 if vp else None,
                 vp.get("iterations_total") if vp else None, vp.get("sequence_speedup") if vp else None,
                 d["roofline"]["kernel"], d["roofline"]["frac"], os.path.basename(f)))
out = ["# Round 1 — bench lines per config (same box; `tools/gpu_round_capture.sh`, `tools/update_profiles.py`)", "",
       "Each line: `python bench.py --config CX [--variant V] [--precond ssor] --steps S --warmup 3` (JSON lines in `r01_lines/`).",
       "`plain` = the same systems of a free-running plain GMRES(m) sequence timed the same way (bench `vs_plain`);",
       "speedup = plain sequence time / recycled sequence time (> 1: recycling pays).  frac = the dominant kernel's",
       "algorithmic bytes / its measured device time over the MEASURED copy peak (6549 GB/s).", "",
       "| config | variant | precond | ms/system | iterations (systems) | plain ms/system | plain iterations | speedup vs plain | dominant kernel | frac | line |",
       "|---|---|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    out.append(f"| {r[0]} | {r[1]} | {r[2]} | {r[3]:.3f} | {r[4]} ({r[5]}) | {'' if r[6] is None else f'{r[6]:.3f}'} | "
               f"{'' if r[7] is None else r[7]} | {'' if r[8] is None else r[8]} | {r[9]} | {r[10]} | {r[11]} |")
open(f"{P}/r01_configs.md", "w").write("\n".join(out) + "\n")

# launch list summary
shutil.copy(f"{cap}/launches.csv", f"{P}/r01_c2_launches.csv")
lrows = list(csv.reader(open(f"{cap}/launches.csv")))
hi = next(i for i, r in enumerate(lrows) if "Kernel Name" in r)
h = lrows[hi]
KN, MV, MU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in lrows[hi + 1:]:
    if len(r) <= MV:
        continue
    m = re.search(r"(k_[A-Za-z0-9_]+(<[^>]*>)?)", r[KN])
    name = m.group(1) if m else r[KN][:40]
    f = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[MU]]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[MV].replace(",", "")) * f
tot = sum(a[1] for a in agg.values())
share = json.loads(open(f"{P}/r01_bench_default_C2.json").read())["roofline"]["share_of_step"]
out = ["# Round 1 — ncu launch list, C2 deflate (bench default), end-of-round kernels", "",
       "Command: `ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file launches.csv python bench.py "
       "--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-vs-plain`",
       "(run after the same bench command exited 0 without ncu; CSV: `r01_c2_launches.csv`).  Cold-cache, serialised per-launch",
       "times: compare SHARES, not absolutes.  One `k_solve_persistent` launch = one whole GMRES solve; `k_cbuild` = the recycle",
       "operator (C = A W, CholQR2 -> Q, R_C^-1) in one cooperative kernel; `k_gram_mma`/`k_gram_reduce`/`k_jacobi`/`k_xm`/`k_inv` =",
       "the two-pass SVD of the snapshot window; `k_fill5_values`/`k_rhs` = the bench's device input generator; `at::` = the bench's",
       f"L2 flush (outside the timed events).  The live bench line (`r01_bench_default_C2.json`) gives the persistent solve {100 * share:.0f} %",
       "of the step (device time incl. host-side gaps between API calls; this list counts kernel time only).", "",
       "| kernel | launches | total us | share of kernel time | avg us |", "|---|---|---|---|---|"]
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.append(f"| {k} | {n} | {t:.1f} | {100 * t / tot:.1f}% | {t / n:.2f} |")
open(f"{P}/r01_c2_launches_summary.md", "w").write("\n".join(out) + "\n")


def ncu_summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h, u, v = rr[0], rr[1], rr[2]
    g = lambda k: (v[h.index(k)], u[h.index(k)]) if k in h else (None, None)
    st = [(h[i], v[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("_not_issued")]
    tsum = sum(float(x[1].replace(",", "")) for x in st if x[1]) or 1.0
    stalls = sorted(((n.replace("smsp__pcsamp_warps_issue_stalled_", ""), 100 * float(x.replace(",", "")) / tsum) for n, x in st),
                    key=lambda t: -t[1])[:5]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
            "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
    return {k: g(k) for k in keys}, stalls


lines = ["# Round 1 — ncu --set full summaries (end of round; .ncu-rep files not committed)", ""]
for rep, what, cmd in ((f"{cap}/persist.ncu-rep", "k_solve_persistent, C2 deflate, system 2 (one whole solve)",
                        "-k regex:k_solve_persistent -s 1 -c 1 ... bench.py --steps 1 --warmup 1"),
                       (f"{cap}/cbuild.ncu-rep", "k_cbuild, C2 deflate, system 8",
                        "-k regex:k_cbuild -s 5 -c 1 ... bench.py --steps 6 --warmup 3")):
    if not os.path.exists(rep):
        continue
    d, s = ncu_summary(rep)
    lines += [f"## {what}", "", f"`ncu --set full --clock-control none --import-source on {cmd} --no-cpu-baseline --no-e2e --no-vs-plain`", "",
              "| metric | value |", "|---|---|"]
    for k, (val, unit) in d.items():
        lines.append(f"| {k} | {val} {unit or ''} |")
    lines.append("| top stall reasons (pc sampling) | " + ", ".join(f"{n} {p:.0f} %" for n, p in s) + " |")
    lines.append("")
open(f"{P}/r01_ncu_full_summaries.md", "w").write("\n".join(lines) + "\n")
print("ok")
