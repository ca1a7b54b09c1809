# Interleaved A/B of kernel library variants on one GPU (tools/perf_attn.py, causal 128K and full 32K):
#   tools/ab.sh TAG VARIANT...   (VARIANT = "tree" for the in-tree library or a tools/exp_lib/NAME)
export PYTHONPATH=$PWD
TAG=$1; shift
OUT=gpurun_out/ab_$TAG; rm -rf $OUT; mkdir -p $OUT
for r in 1 2; do
 for v in "$@"; do
  if [ $v = tree ]; then unset BB_LIB_PATH; else export BB_LIB_PATH=tools/exp_lib/$v/libburst_b200.so; fi
  echo "== $v causal" >> $OUT/perf.log; timeout 60 python tools/perf_attn.py >> $OUT/perf.log 2>&1
  echo "== $v full32k" >> $OUT/perf.log; timeout 60 python tools/perf_attn.py --n 32768 --mask full >> $OUT/perf.log 2>&1
 done
done
