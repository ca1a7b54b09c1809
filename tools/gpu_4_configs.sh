# 4 B200: cfg4 (512K, GQA 32/8, SWA ∩ documents, block_striped) with both backward passes, and the
# 1M-token causal headline on the two-level 2x2 ring plan
export PYTHONPATH=$PWD
mkdir -p gpurun_out/cfg4_4
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531"
for bw in burst_backward ring_backward; do
  timeout 900 $R bench.py --gpus 4 --steps 3 --warmup 3 --seq 524288 --kv-heads 8 --mask swa_doc --layout block_striped \
    --backward $bw --no-cpu --no-lmhead --no-1m > gpurun_out/cfg4_4/cfg4_$bw.json 2> gpurun_out/cfg4_4/cfg4_$bw.err
done
timeout 900 $R bench.py --gpus 4 --steps 2 --warmup 2 --seq 1048576 --topology 2x2 --no-cpu --no-lmhead --no-e2e \
  > gpurun_out/cfg4_4/cfg3_2x2.json 2> gpurun_out/cfg4_4/cfg3_2x2.err
