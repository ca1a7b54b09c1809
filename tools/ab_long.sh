# A/B of library variants on a long causal step (512K rows, 8 heads, one GPU)
export PYTHONPATH=$PWD
TAG=$1; shift
OUT=gpurun_out/abl_$TAG; rm -rf $OUT; mkdir -p $OUT
for r in 1 2; do
for v in "$@"; do
  if [ $v = tree ]; then unset BB_LIB_PATH; else export BB_LIB_PATH=tools/exp_lib/$v/libburst_b200.so; fi
  echo "== $v" >> $OUT/perf.log; timeout 300 python tools/perf_attn.py --n 524288 --heads 8 --iters 1 >> $OUT/perf.log 2>&1
done
done
