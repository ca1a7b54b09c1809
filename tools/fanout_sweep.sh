export PYTHONPATH=$PWD
for f in 1 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N:-2} --master-addr 127.0.0.1 --master-port 2951$f \
    bench.py --gpus ${N:-2} --steps 2 --warmup 3 --no-e2e --ce-fanout $f > gpurun_out/fan$f.json 2> gpurun_out/fan$f.err
  echo "fanout $f exit $?" >> gpurun_out/fan.log
done
