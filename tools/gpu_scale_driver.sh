# the driver's scaling settings on this box: default bench line at N=4 and N=2 with --steps 20 --warmup 5
export PYTHONPATH=$PWD
mkdir -p gpurun_out/scale20
for N in 4 2; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N \
    bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/scale20/bench_${N}gpu.json 2> gpurun_out/scale20/bench_${N}gpu.err
done
