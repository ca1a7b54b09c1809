"""Per-phase clock64 timeline of one backward CTA (BB_PROBE=1)."""
import ctypes, os, sys
os.environ["BB_PROBE"] = "1"
import numpy as np, torch
sys.argv += []
from paper_2509_19836_b200 import _native as N
import runpy
sys.argv = ["perf_attn.py", "--n", "32768", "--heads", "8", "--iters", "1", "--mask", "full"]
runpy.run_path("tools/perf_attn.py", run_name="__main__")
buf = np.zeros(4096, dtype=np.int64)
N.check(N.load().bb_debug_probe(buf.ctypes.data, 4096))
t = buf.reshape(128, 32)[:16]
base = t[t > 0].min()
names = {24: "c:top", 0: "ld:q_empty?", 1: "ld:q_empty ok", 2: "ld:do_empty ok", 4: "mma:start", 5: "mma:q_full", 6: "mma:S issued", 7: "mma:dq_free", 8: "mma:p_full", 9: "mma:ds_full",
         16: "c:start", 17: "c:s_full", 18: "c:P done", 19: "c:dp_full", 20: "c:dS done", 21: "c:dq_full", 22: "c:dq drained", 23: "c:end"}
for it in range(16):
    row = " ".join(f"{names[s]}={t[it, s]-base}" for s in sorted(names) if t[it, s] > 0)
    print(it, row)
