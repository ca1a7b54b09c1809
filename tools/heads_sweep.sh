export PYTHONPATH=$PWD
mkdir -p gpurun_out/heads
for h in 1 4 8 16 32 64; do timeout 60 python tools/perf_attn.py --n 32768 --mask full --heads $h >> gpurun_out/heads/full32k.log 2>&1; done
for h in 8 32; do timeout 90 python tools/perf_attn.py --n 131072 --heads $h >> gpurun_out/heads/causal128k.log 2>&1; done
