# round-end state on 4 B200: multi-GPU parity tests (incl. 1M tokens), then the default bench line at N=2 and N=4
export PYTHONPATH=$PWD
mkdir -p gpurun_out/final4
timeout 2400 python -m pytest tests/test_ring_multigpu.py -m gpu -q -p no:cacheprovider > gpurun_out/final4/multigpu_tests.txt 2>&1; echo "exit $?" >> gpurun_out/final4/multigpu_tests.txt
for N in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N \
    bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/final4/bench_${N}gpu.json 2> gpurun_out/final4/bench_${N}gpu.err
  echo "bench $N exit $?" >> gpurun_out/final4/multigpu_tests.txt
done
