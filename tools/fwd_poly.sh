# forward exp-split variants (tools/exp_lib/polyN, BB_FWD_POLY=N) vs the in-tree library, plus a probe timeline
export PYTHONPATH=$PWD
mkdir -p gpurun_out/fwdh
timeout 100 python tools/probe_fwd.py > gpurun_out/fwdh/probe.log 2>&1
for r in 1 2; do
 for v in new poly2 poly3 poly4; do
  if [ $v = new ]; then unset BB_LIB_PATH; else export BB_LIB_PATH=tools/exp_lib/$v/libburst_b200.so; fi
  echo "== $v causal" >> gpurun_out/fwdh/poly.log
  timeout 60 python tools/perf_attn.py >> gpurun_out/fwdh/poly.log 2>&1
  echo "== $v full32k" >> gpurun_out/fwdh/poly.log
  timeout 60 python tools/perf_attn.py --n 32768 --mask full >> gpurun_out/fwdh/poly.log 2>&1
 done
done
