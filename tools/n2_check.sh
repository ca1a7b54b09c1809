# 2-GPU round check: GPU tests touching the ring helpers, multi-GPU ring parity, a 2-GPU bench line, the gap trace
export PYTHONPATH=$PWD
mkdir -p gpurun_out/n2
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_layer_gpu.py tests/test_parity_gpu.py tests/test_ring_multigpu.py -x -q > gpurun_out/n2/tests.log 2>&1; echo "exit $?" >> gpurun_out/n2/tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/n2/bench.json 2> gpurun_out/n2/bench.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 tools/ring_gaps.py > gpurun_out/n2/gaps.log 2>&1
