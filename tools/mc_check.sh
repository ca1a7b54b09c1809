export PYTHONPATH=$PWD
for rep in 1 2 3; do timeout 200 python tools/bwd_heads_check.py > gpurun_out/mc_hc$rep.log 2>&1; echo "heads_check $rep exit $?" >> gpurun_out/mc.log; done
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider > gpurun_out/mc_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/mc.log
for v in mc0 mc1; do echo "== $v" >> gpurun_out/mc.log; BB_LIB_PATH=paper_2509_19836_b200/_lib/variants/lib_$v.so python tools/perf_attn.py --n 32768 --heads 32 --mask full 2>&1 | grep bwd >> gpurun_out/mc.log; BB_LIB_PATH=paper_2509_19836_b200/_lib/variants/lib_$v.so python tools/perf_attn.py 2>&1 | grep bwd >> gpurun_out/mc.log; done
