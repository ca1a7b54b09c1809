# usage: bash tools/prof_run.sh <kernel-regex> <args for perf_attn.py...>
# plain run first (must exit 0), then one ncu --set full capture of the named kernel
export PYTHONPATH=$PWD
K=$1; shift
python tools/perf_attn.py --iters 1 "$@" > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_$K -f \
    python tools/perf_attn.py --iters 1 "$@" > gpurun_out/prof_ncu.log 2>&1
echo "exit $?" >> gpurun_out/prof_ncu.log
