export PYTHONPATH=$PWD
for v in "$@"; do
  echo "== $v" >> gpurun_out/bvariants.log
  BB_LIB_PATH=paper_2509_19836_b200/_lib/variants/lib_$v.so python tools/perf_attn.py --n 32768 --heads 32 --mask full 2>&1 | grep bwd >> gpurun_out/bvariants.log
  BB_LIB_PATH=paper_2509_19836_b200/_lib/variants/lib_$v.so python tools/perf_attn.py 2>&1 | grep bwd >> gpurun_out/bvariants.log
done
