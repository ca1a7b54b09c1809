# A/B of library variants on causal attention at several lengths (tools/exp_lib/NAME or "tree")
export PYTHONPATH=$PWD
TAG=$1; shift
OUT=gpurun_out/abc_$TAG; rm -rf $OUT; mkdir -p $OUT
for v in "$@"; do
  if [ $v = tree ]; then unset BB_LIB_PATH; else export BB_LIB_PATH=tools/exp_lib/$v/libburst_b200.so; fi
  for n in 16384 32768 131072; do
    echo "== $v causal $n" >> $OUT/perf.log; timeout 120 python tools/perf_attn.py --n $n >> $OUT/perf.log 2>&1
  done
done
