# One-GPU sweep of the bench over the SURVEY configs (JSON lines into gpurun_out/sweep_cfg*.json)
export PYTHONPATH=$PWD
run() { tag=$1; shift; timeout 600 python bench.py --no-cpu "$@" > gpurun_out/sweep_$tag.json 2> gpurun_out/sweep_$tag.err; \
  python -c "import json; d=json.loads(open('gpurun_out/sweep_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['value'],1), (d.get('e2e') or {}).get('value'), d['config']['workload'][:110], d['clocks']['sm_mhz'])"; }
run cfg2 
run cfg2_full --mask full
run cfg2_d64 --head-dim 64 --heads 64
run cfg2_ring --backward ring_backward
run cfg4 --seq 524288 --kv-heads 8 --mask swa_doc --layout block_striped --steps 3
run cfg2_window --mask window --window 32768
