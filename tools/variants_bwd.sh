export PYTHONPATH=$PWD
for v in "$@"; do
  echo "== $v" >> gpurun_out/variants_bwd.log
  BB_LIB_PATH=paper_2509_19836_b200/_lib/variants/lib_$v.so timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k "bwd" -x -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/variants_bwd.log
  BB_LIB_PATH=paper_2509_19836_b200/_lib/variants/lib_$v.so python tools/perf_attn.py >> gpurun_out/variants_bwd.log 2>&1
  BB_LIB_PATH=paper_2509_19836_b200/_lib/variants/lib_$v.so python tools/perf_attn.py --n 32768 --mask full >> gpurun_out/variants_bwd.log 2>&1
done
