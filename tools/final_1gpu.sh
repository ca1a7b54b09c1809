# Round-end state on one B200: full GPU suite, smoke, default bench line
export PYTHONPATH=$PWD
mkdir -p gpurun_out/final1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final1/gpu_suite.txt 2>&1; echo "exit $?" >> gpurun_out/final1/gpu_suite.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final1/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/final1/bench.json 2> gpurun_out/final1/bench.err
