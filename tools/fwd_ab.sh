# A/B of the forward kernel: tools/exp_lib/base (previous build) vs the in-tree library
export PYTHONPATH=$PWD
rm -rf gpurun_out/fwdh; mkdir -p gpurun_out/fwdh
timeout 60 python tools/perf_attn.py --n 32768 --heads 8 --mask full --iters 2 > gpurun_out/fwdh/smoke.log 2>&1 || { echo "smoke failed $?" >> gpurun_out/fwdh/smoke.log; exit 1; }
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_mask_exact_gpu.py tests/test_layer_gpu.py -x -q ${TESTK:+-k "$TESTK"} > gpurun_out/fwdh/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/fwdh/tests.log
for r in 1 2; do
 for v in base new; do
  if [ $v = base ]; then export BB_LIB_PATH=tools/exp_lib/base/libburst_b200.so; else unset BB_LIB_PATH; fi
  echo "== $v causal" >> gpurun_out/fwdh/perf.log
  timeout 60 python tools/perf_attn.py >> gpurun_out/fwdh/perf.log 2>&1
  echo "== $v full32k" >> gpurun_out/fwdh/perf.log
  timeout 60 python tools/perf_attn.py --n 32768 --mask full >> gpurun_out/fwdh/perf.log 2>&1
 done
done
