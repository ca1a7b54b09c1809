"""Split an ncu SASS source-page CSV of a warp-specialised kernel into role regions at its
USETMAXREG instructions and print stall samples per region plus the hottest instructions.

    ncu -i rep --page source --csv --print-source sass > x.csv; python tools/ncu_regions.py x.csv [--top 15]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 15
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
S = ix["Warp Stall Sampling (All Samples)"]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
region = "prologue"
seg = []
for r in data:
    src = r[ix["Source"]]
    if "USETMAXREG" in src:
        region = src.strip().split()[-1].rstrip(";") if "DEALLOC" not in src else "dealloc " + src.strip().split()[-1].rstrip(";")
        region = ("alloc " if "TRY_ALLOC" in src else "") + region
    if "EXIT" in src and region != "prologue":
        seg.append(("exit", r))
        continue
    seg.append((region, r))
tot = Counter()
rc = {}
for k, r in seg:
    s = int(r[S] or 0)
    tot[k] += s
    c = rc.setdefault(k, Counter())
    for h in reasons:
        c[h[6:]] += int(r[ix[h]] or 0)
T = sum(tot.values())
for k, v in tot.most_common():
    print(f"{k:24s} {v:8d} {100 * v / T:5.1f}%  " + ", ".join(f"{a} {100 * b / max(v, 1):.0f}%" for a, b in rc[k].most_common(5)))
    ins = sorted(((int(r[S] or 0), r[ix["Address"]][-5:], r[ix["Source"]].strip()[:58],
                   sorted(((int(r[ix[h]] or 0), h[6:]) for h in reasons), reverse=True)[:2]) for kk, r in seg if kk == k),
                 reverse=True)[:top]
    for x in ins:
        if x[0] > 0:
            print(f"    {x[0]:7d} {x[1]} {x[2]:58s} {x[3]}")
