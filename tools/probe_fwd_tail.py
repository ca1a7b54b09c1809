import os, sys, runpy
os.environ["BB_PROBE"] = "1"
os.environ["BB_LIB_PATH"] = "tools/exp_lib/probetail/libburst_b200.so"
import numpy as np
from paper_2509_19836_b200 import _native as N
sys.argv = ["perf_attn.py", "--n", "16384", "--heads", "32", "--iters", "1", "--mask", "causal"]
runpy.run_path("tools/perf_attn.py", run_name="__main__")
buf = np.zeros(4096, dtype=np.int64)
N.check(N.load().bb_debug_probe(buf.ctypes.data, 4096))
t = buf[512:1024].reshape(16, 32)
base = t[t > 0].min()
for it in range(15, -1, -1):
    r = t[it]
    print(f"tile j_hi-1-{it:2d}: q0 S?={r[16]-base:7d} S={r[17]-base:7d} P={r[19]-base:7d} | q1 S?={r[24]-base:7d} S={r[25]-base:7d} P={r[27]-base:7d}")
