"""Aggregate an ncu `--page source --csv --print-source cuda,sass` dump per CUDA source line:
warp-stall samples and their top reasons (the SASS rows under each source row).

    ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [--top 40]
"""
import csv
import sys
from collections import Counter, defaultdict

path = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
f = None
line = None
src = {}
samples = Counter()
reasons = defaultdict(Counter)
hdr = None
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = True
        stall_cols = [(i, h) for i, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h]
        samp = r.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= samp:
        continue
    if r[0]:
        line = (f, int(r[0]))
        src[line] = r[1].strip()
        continue
    try:
        s = int(r[samp])
    except ValueError:
        continue
    samples[line] += s
    for i, h in stall_cols:
        try:
            reasons[line][h[6:]] += int(r[i])
        except ValueError:
            pass
tot = sum(samples.values())
print("total samples", tot)
for ln, s in samples.most_common(top):
    rs = ", ".join(f"{k} {100 * v / max(s, 1):.0f}%" for k, v in reasons[ln].most_common(3))
    print(f"{100 * s / tot:5.1f}% {ln[0]}:{ln[1]:<5d} {src.get(ln, '')[:70]:70s} {rs}")
