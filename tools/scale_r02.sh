# Round-2 multi-GPU runs (one box, N = $1 GPUs): cfg2 128K and the 1M-token headline, CE ring.
export PYTHONPATH=$PWD
N=${1:-4}
mkdir -p gpurun_out/r02_scaling; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29537 tools/ring_check.py > gpurun_out/r02_scaling/ring_check_$N.log 2>&1; echo "ring_check rc=$?"
run() {  # name, extra bench args
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --gpus $N "${@:2}" > gpurun_out/r02_scaling/$1.json 2> gpurun_out/r02_scaling/$1.err
  echo "$1 rc=$?"
}
run scale${N}_128k --steps 5 --warmup 3 --no-lmhead
run scale${N}_1m --seq 1048576 --steps 3 --warmup 3 --no-e2e --no-lmhead
if [ $N -eq 4 ]; then run scale4_1m_2x2 --seq 1048576 --topology 2x2 --steps 2 --warmup 1 --no-e2e --no-lmhead; fi
