# cfg4 on 4 GPUs: GQA 32q/8kv, 512K tokens, sliding window 32K AND 128K causal documents
# (block mask), block_striped layout; burst and ring backward over the copy-engine ring
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for bw in ring_backward burst_backward; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 4 --steps 3 --warmup 3 --seq 524288 --kv-heads 8 --mask swa_doc --layout block_striped \
    --backward $bw --no-e2e > gpurun_out/cfg4_n4_$bw.json 2> gpurun_out/cfg4_n4_$bw.err
  echo "cfg4 $bw exit $?" >> gpurun_out/cfg4.log
done
