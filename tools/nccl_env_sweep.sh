# N-GPU bench under a few NCCL settings (P2P channel count / chunk size): bash tools/nccl_env_sweep.sh N
export PYTHONPATH=$PWD
N=${1:-4}
run() {
  tag=$1; shift
  env "$@" timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 200)) bench.py --gpus $N --no-e2e --no-cpu > gpurun_out/sweep_$tag.json 2> gpurun_out/sweep_$tag.err
  python -c "import json; d=json.loads(open('gpurun_out/sweep_$tag.json').read().strip().splitlines()[-1]); o=d['ring_overlap']; print('$tag', round(d['value'],1), round(o['comm_alone_ms'],2), round(o['exposed_comm_ms'],2), round(o['hidden_frac'],2))"
}
run default
run ch2 NCCL_MAX_NCHANNELS=2
run ch8 NCCL_MIN_NCHANNELS=8
run chunk1m NCCL_P2P_NVL_CHUNKSIZE=1048576
