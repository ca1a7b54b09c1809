# A/B of library variants on full-mask backward (where every key tile sees every query tile)
export PYTHONPATH=$PWD
TAG=$1; shift
OUT=gpurun_out/abf_$TAG; rm -rf $OUT; mkdir -p $OUT
for r in 1 2; do
for v in "$@"; do
  if [ $v = tree ]; then unset BB_LIB_PATH; else export BB_LIB_PATH=tools/exp_lib/$v/libburst_b200.so; fi
  echo "== $v full 32K" >> $OUT/perf.log; timeout 120 python tools/perf_attn.py --n 32768 --mask full >> $OUT/perf.log 2>&1
  echo "== $v full 256K h8" >> $OUT/perf.log; timeout 300 python tools/perf_attn.py --n 262144 --heads 8 --mask full --iters 1 >> $OUT/perf.log 2>&1
  echo "== $v causal 128K" >> $OUT/perf.log; timeout 120 python tools/perf_attn.py >> $OUT/perf.log 2>&1
done
done
