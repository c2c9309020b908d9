"""Static SASS instruction counts per kernel of librg.so (profiles/r02/sass_summary.md): where the FP64
tensor-core path (DMMA), the 1-D bulk copies (UBLKCP), tensor-map TMA loads (UTMALDG) and mbarrier
operations (SYNCS) are.  python tools/sass_summary.py [lib] [out.md]"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1807_09467_b200/lib/librg.so"
out_md = sys.argv[2] if len(sys.argv) > 2 else "profiles/r02/sass_summary.md"
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
rows = {}
for f in re.split(r"\n\s*Function : ", txt)[1:]:
    name = f.split("\n", 1)[0].strip()
    m = re.search(r"(k_[a-z0-9_]+)", name)
    short = m.group(1) if m else name[:40]
    tm = re.search(r"ILi(\d+)E(?:Li(\d+)E)?(?:Li(\d+)E)?", name)
    if tm:
        short += "<" + ",".join(x for x in tm.groups() if x) + ">"

    def c(pat):
        return len(re.findall(pat, f))
    row = (c(r"\bDMMA\b"), c(r"\bUBLKCP\b"), c(r"\bUTMALDG\b"), c(r"\bSYNCS\."), c(r"\bDFMA\b"), c(r"\bLDG\b"),
           c(r"\bLDS\b"), c(r"\bBAR\b"), c(r"\bRED\.|\bATOM"))
    rows.setdefault(short, row)  # one line per kernel (instantiations per variant family collapse)
out = ["| kernel | DMMA | UBLKCP (cp.async.bulk) | UTMALDG (tensor TMA) | SYNCS (mbarrier) | DFMA | LDG | LDS | BAR | ATOM/RED |",
       "|---|---|---|---|---|---|---|---|---|---|"]
for k in sorted(rows):
    out.append("| `%s` | " % k + " | ".join(str(v) for v in rows[k]) + " |")
hdr = ("# SASS instruction summary of librg.so (`cuobjdump -sass`, sm_100a)\n\n"
       "Static instruction counts per kernel (not executed counts).  No tcgen05 (UTC*) instructions: sm_100a\n"
       "has no f64 kind of tcgen05.mma, so the FP64 tensor path is DMMA (mma.sync .f64).\n"
       "Regenerate: `python tools/sass_summary.py`.\n\n")
open(out_md, "w").write(hdr + "\n".join(out) + "\n")
print("\n".join(out))
