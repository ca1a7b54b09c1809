"""Decode Volta+ SASS control codes (stall / yield / barriers) from cuobjdump -sass text and
sum the static stall cycles over a window.   python tools/sass_ctrl.py file.sass START END"""
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
a, b = int(sys.argv[2], 0), int(sys.argv[3], 0)
ins = []
i = 0
while i < len(lines) - 1:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* 0x([0-9a-f]{16}) \*/", lines[i])
    if m:
        m2 = re.search(r"/\* 0x([0-9a-f]{16}) \*/", lines[i + 1])
        if m2:
            hi = int(m2.group(1), 16)
            ins.append((int(m.group(1), 16), m.group(2).strip(), (hi >> 41) & 0xF, (hi >> 45) & 1,
                        (hi >> 46) & 7, (hi >> 49) & 7, (hi >> 52) & 0x3F))
            i += 2
            continue
    i += 1
sel = [x for x in ins if a <= x[0] <= b]
tot = sum(x[2] for x in sel)
for x in sel:
    if "-v" in sys.argv:
        print(f"{x[0]:06x} st={x[2]:2d} y={x[3]} wb={x[4]} rb={x[5]} wm={x[6]:06b}  {x[1][:70]}")
print(f"{len(sel)} instructions, static stall sum {tot} cycles, MUFU {sum('MUFU' in x[1] for x in sel)}")
