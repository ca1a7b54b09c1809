"""Count local-memory spills (STL/LDL) per setmaxnreg region of a kernel in a cubin/object.
    python tools/sass_spills.py obj.o <kernel-name-substring>"""
import re
import subprocess
import sys
from collections import Counter

sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
cur, region, c = None, "prologue", Counter()
for l in sass.split("\n"):
    m = re.search(r"Function : (\S+)", l)
    if m:
        cur, region = m.group(1), "prologue"
        continue
    if cur is None or sys.argv[2] not in cur:
        continue
    if "USETMAXREG" in l:
        region = l.strip().split(";")[0].split()[-1]
    for op in ("STL", "LDL"):
        if re.search(r"\b" + op + r"\b", l):
            c[(region, op)] += 1
for k, v in sorted(c.items()):
    print(k, v)
