nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
for t in test_gemm test_fwd_single test_fwd_two test_bwd test_lmhead; do
  timeout 240 python -m pytest tests/test_kernels_gpu.py -q -k $t -x -p no:cacheprovider > gpurun_out/k_$t.log 2>&1
  echo "$t exit $?" >> gpurun_out/summary.txt
done
