# A/B of library variants: causal 128K (32 heads) and causal 512K (8 heads), one GPU, interleaved twice
export PYTHONPATH=$PWD
TAG=$1; shift
OUT=gpurun_out/abm_$TAG; rm -rf $OUT; mkdir -p $OUT
for r in 1 2; do
for v in "$@"; do
  if [ $v = tree ]; then unset BB_LIB_PATH; else export BB_LIB_PATH=tools/exp_lib/$v/libburst_b200.so; fi
  echo "== $v 128K" >> $OUT/perf.log; timeout 120 python tools/perf_attn.py >> $OUT/perf.log 2>&1
  echo "== $v 512K" >> $OUT/perf.log; timeout 300 python tools/perf_attn.py --n 524288 --heads 8 --iters 1 >> $OUT/perf.log 2>&1
done
done
