"""Per-phase clock64 timeline of one backward CTA (BB_PROBE=1): CTA (0,0), first 16 tiles.
Slot meanings follow BB_PROBE(n) in csrc/bb_attn_bwd.cu."""
import os
import runpy
import sys

os.environ["BB_PROBE"] = "1"
# the product library compiles the probes out: build `python tools/variant.py probes BB_WITH_PROBES`
os.environ.setdefault("BB_LIB_PATH", "tools/exp_lib/probes/libburst_b200.so")
import numpy as np

from paper_2509_19836_b200 import _native as N

sys.argv = ["perf_attn.py", "--n", "32768", "--heads", "8", "--iters", "1", "--mask", "full"]
runpy.run_path("tools/perf_attn.py", run_name="__main__")
buf = np.zeros(4096, dtype=np.int64)
N.check(N.load().bb_debug_probe(buf.ctypes.data, 4096))
t = buf.reshape(128, 32)[:16]
base = t[t > 0].min()
names = {0: "ld:q_empty?", 1: "ld:q_empty ok", 2: "ld:do_empty ok",
         4: "mma:top", 8: "mma:p_full ok", 5: "mma:dV+S issued", 9: "mma:ds_full ok", 6: "mma:do_full ok",
         7: "mma:dq_free ok", 10: "mma:dK+dQ issued", 11: "mma:dP issued",
         24: "c0:top", 16: "c0:pre-S", 17: "c0:S ok", 18: "c0:P done", 19: "c0:dP ok", 20: "c0:dS done", 23: "c0:end",
         30: "c0:pre-dP", 31: "c1:pre-dP", 25: "c1:top", 26: "c1:S ok", 27: "c1:P done", 28: "c1:dP ok", 29: "c1:dS done",
         21: "dq:top", 22: "dq:drained"}
order = [0, 1, 2, 4, 8, 5, 9, 10, 6, 7, 11, 24, 16, 17, 18, 30, 19, 20, 23, 25, 26, 27, 31, 28, 29, 21, 22]
for it in range(16):
    print(it, " ".join(f"{names[s]}={t[it, s] - base}" for s in order if t[it, s] > 0))
