"""Per-phase clock64 timeline of one forward CTA (BB_PROBE=1)."""
import os, sys, runpy
os.environ["BB_PROBE"] = "1"
# the product library compiles the probes out: build `python tools/variant.py probes BB_WITH_PROBES`
os.environ.setdefault("BB_LIB_PATH", "tools/exp_lib/probes/libburst_b200.so")
import numpy as np
from paper_2509_19836_b200 import _native as N
sys.argv = ["perf_attn.py", "--n", "32768", "--heads", "8", "--iters", "1", "--mask", "full"] + sys.argv[1:]
runpy.run_path("tools/perf_attn.py", run_name="__main__")
buf = np.zeros(4096, dtype=np.int64)
N.check(N.load().bb_debug_probe(buf.ctypes.data, 4096))
t = buf[512:1024].reshape(16, 32)
base = t[t > 0].min()
names = {20: "s0:exp", 21: "s0:stw", 22: "s0:bits", 23: "s0:ldS", 28: "s1:exp", 29: "s1:stw", 30: "s1:bits", 31: "s1:ldS", 0: "ld:K?", 1: "ld:K", 2: "ld:V?", 3: "ld:V", 4: "m:K?", 5: "m:K", 6: "m:P0?", 7: "m:P0", 8: "m:P1?", 9: "m:P1",
         16: "s0:S?", 17: "s0:S", 18: "s0:pv", 19: "s0:P", 24: "s1:S?", 25: "s1:S", 26: "s1:pv", 27: "s1:P"}
for it in range(16):
    print(it, " ".join(f"{names[s]}={t[it, s]-base}" for s in sorted(names) if t[it, s] > 0))
