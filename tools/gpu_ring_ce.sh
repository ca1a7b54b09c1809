# multi-GPU ring on N GPUs (gpurun --gpus N): parity of both transports, then bench lines
N=${1:-2}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
BB_RING_LOG_DIR=gpurun_out timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  tools/ring_check.py > gpurun_out/rc$N.log 2>&1; echo "ring_check exit $?" >> gpurun_out/rc$N.log
for tr in ${TRANSPORTS:-ce collective}; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus $N --steps 3 --warmup 3 --transport $tr ${BENCH_EXTRA} > gpurun_out/b${N}_$tr.json 2> gpurun_out/b${N}_$tr.err
  echo "bench $tr exit $?" >> gpurun_out/rc$N.log
done
