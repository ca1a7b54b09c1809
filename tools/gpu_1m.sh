# 4 GPUs: ring parity (both transports + autograd), then 1M-token causal bench lines for the
# two-level 2x2 ring and the flat 1x4 ring (copy-engine transport)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
BB_RING_LOG_DIR=gpurun_out timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29511 tools/ring_check.py > gpurun_out/rc4.log 2>&1; echo "ring_check exit $?" >> gpurun_out/rc4.log
for topo in 2x2 1x4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 4 --steps 2 --warmup 3 --seq 1048576 --topology $topo --no-e2e > gpurun_out/b4_1m_$topo.json 2> gpurun_out/b4_1m_$topo.err
  echo "bench $topo exit $?" >> gpurun_out/rc4.log
done
