# Round profile: default bench line, then (same command lines, after they exited 0) the ncu
# launch list and one --set full capture of each attention kernel.
export PYTHONPATH=$PWD
R=${1:-r01}
python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err || exit 1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_$R.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv $CMD > gpurun_out/ncu_launch_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 1 -c 1 -o gpurun_out/prof_bwd_$R -f $CMD > gpurun_out/ncu_bwd_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/prof_fwd_$R -f $CMD > gpurun_out/ncu_fwd_$R.log 2>&1
echo "exit $?" >> gpurun_out/ncu_launch_$R.log
