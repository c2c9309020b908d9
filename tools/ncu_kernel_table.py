"""Summarise an ncu CSV (gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum) of
tools/prof_multi.py C3/C4/C5 runs into a per-config, per-kernel DRAM-bandwidth table (markdown).
The config of each launch is inferred from the SpMV format kernel that precedes it."""
import collections
import csv
import re
import statistics
import sys

path = sys.argv[1]
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ID, KN, MN, MV = h.index('ID'), h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= MV:
        continue
    m = re.search(r'(k_[A-Za-z0-9_]+(<[^>]*>)?)', r[KN])
    d = launch.setdefault(r[ID], {"name": m.group(1) if m else r[KN][:40]})
    d[r[MN]] = float(r[MV].replace(',', ''))
segname = {"k_spmv_sell": "C3", "k_spmv_csr<1>": "C4", "k_spmv_bsr_tma": "C5"}
seg, out = None, collections.OrderedDict()
for d in launch.values():
    n = d["name"]
    if n in segname:
        seg = segname[n]
    t = d.get("gpu__time_duration.sum", 0.0)
    by = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    if by < 65536:  # a no-op launch (the device state said "nothing to do"): not a bandwidth sample
        continue
    out.setdefault((seg or "?", n), []).append((t, by))
peak_copy, peak_read = float(sys.argv[2]), float(sys.argv[3])
print("| config | kernel | launches | total ms | DRAM GB | DRAM GB/s | median launch GB/s | / copy peak | / read peak |")
print("|---|---|---|---|---|---|---|---|---|")
for (s, n), a in out.items():
    T = sum(x[0] for x in a) * 1e-9
    B = sum(x[1] for x in a)
    g = B / T / 1e9 if T else 0.0
    med = statistics.median([x[1] / (x[0] * 1e-9) / 1e9 for x in a if x[0] > 0])
    print(f"| {s} | {n} | {len(a)} | {T * 1e3:.2f} | {B / 1e9:.2f} | {g:.0f} | {med:.0f} | {g / peak_copy:.2f} | {g / peak_read:.2f} |")
