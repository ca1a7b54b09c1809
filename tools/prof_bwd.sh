# ncu capture of one attention kernel on a mid-size case (after the plain run exits 0)
#   tools/prof_bwd.sh TAG [attn_bwd|attn_fwd] [perf_attn args...]
export PYTHONPATH=$PWD
TAG=$1; KER=${2:-attn_bwd}; shift 2
ARGS=${@:---n 32768 --heads 8 --mask full --iters 2}
CMD="python tools/perf_attn.py $ARGS"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KER -s 1 -c 1 -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/ncu_$TAG.log
