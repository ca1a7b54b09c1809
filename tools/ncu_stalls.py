"""Summarise an ncu source-page CSV (ncu -i rep --page source --csv --print-source sass):
stall samples per reason over the whole kernel and over the hottest instruction windows.

    python tools/ncu_stalls.py src.csv [--top 40]
"""
import csv
import sys
from collections import Counter

path = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for r in data:
    for h in reasons:
        try:
            tot[h] += int(r[ix[h]])
        except ValueError:
            pass
S = sum(tot.values())
print("total samples", S)
for h, v in tot.most_common():
    if v:
        print(f"  {h:28s} {v:8d} {100 * v / S:5.1f}%")
print("\nhottest instructions:")
hot = sorted(data, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:top]
for r in hot:
    reasons_r = sorted(((int(r[ix[h]] or 0), h[6:]) for h in reasons), reverse=True)[:3]
    print(f"{r[ix['Address']][-5:]} {int(r[ix['Warp Stall Sampling (All Samples)']]):6d}  {r[ix['Source']].strip()[:60]:60s} {reasons_r}")

# per-region breakdown: contiguous address windows around MUFU.EX2 clusters (the exp pass)
addrs = [int(r[ix["Address"]], 16) for r in data]
mufu = [i for i, r in enumerate(data) if "MUFU.EX2" in r[ix["Source"]]]
if mufu and "--regions" in sys.argv:
    clusters = []
    start = prev = mufu[0]
    for i in mufu[1:]:
        if i - prev > 40:
            clusters.append((start, prev))
            start = i
        prev = i
    clusters.append((start, prev))
    for a, b in clusters:
        seg = data[a:b + 1]
        c = Counter()
        n_ins = len(seg)
        for r in seg:
            for h in reasons:
                c[h[6:]] += int(r[ix[h]] or 0)
        s = sum(c.values())
        ex = sum(int(r[ix["Instructions Executed"]] or 0) for r in seg)
        print(f"MUFU cluster {a}-{b}: {n_ins} instr, {sum('MUFU' in r[ix['Source']] for r in seg)} MUFU, warp-instr executed {ex}, samples {s}:",
              ", ".join(f"{k} {100 * v / max(s, 1):.0f}%" for k, v in c.most_common(6)))
