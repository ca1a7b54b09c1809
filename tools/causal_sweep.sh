# forward / backward rate of causal vs full masks over sequence length (32 heads, one GPU)
export PYTHONPATH=$PWD
mkdir -p gpurun_out/cs
for n in 16384 32768 65536 131072; do
  for m in causal full; do
    echo "== $n $m" >> gpurun_out/cs/sweep.log
    timeout 120 python tools/perf_attn.py --n $n --mask $m >> gpurun_out/cs/sweep.log 2>&1
  done
done
