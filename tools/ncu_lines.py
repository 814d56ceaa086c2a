"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export per CUDA source line:
warp-stall samples (all / not-issued) and the top stall reasons.  Usage:
    ncu -i rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top_n]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
fname = None
hdr = None
agg = defaultdict(lambda: defaultdict(float))
src = {}
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0] != "":
        cur = (fname, int(r[0]))
        src[cur] = r[1]
        continue
    d = dict(zip(hdr[2:], r[2:]))
    a = agg[cur]
    for k, v in d.items():
        if k.startswith("stall_") or k in ("Warp Stall Sampling (All Samples)",
                                           "Warp Stall Sampling (Not-issued Samples)",
                                           "Instructions Executed"):
            try:
                a[k] += float(v)
            except ValueError:
                pass
tot = sum(a["Warp Stall Sampling (All Samples)"] for a in agg.values())
print(f"total samples {tot:.0f}")
order = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])
for (f, ln), a in order[:top]:
    s = a["Warp Stall Sampling (All Samples)"]
    st = sorted(((v, k) for k, v in a.items() if k.startswith("stall_") and "Not Issued" not in k),
                reverse=True)[:3]
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5} {src[(f, ln)][:60]:60s} "
          + " ".join(f"{k[6:]}={100 * v / max(s, 1):.0f}%" for v, k in st))
