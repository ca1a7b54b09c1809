# Round-2 ncu captures of the bench command (each after the plain run exits 0):
# launch list (per-kernel device time) and one --set full capture each of attn_bwd / attn_fwd.
export PYTHONPATH=$PWD
R=${1:-r02}
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-lmhead"
$CMD > gpurun_out/plain_$R.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv $CMD > gpurun_out/ncu_launch_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 1 -c 1 -o gpurun_out/prof_bwd_$R -f $CMD > gpurun_out/ncu_bwd_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/prof_fwd_$R -f $CMD > gpurun_out/ncu_fwd_$R.log 2>&1
echo "exit $?" >> gpurun_out/ncu_launch_$R.log
