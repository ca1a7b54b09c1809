export PYTHONPATH=$PWD
for tr in ce collective ce; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus 4 --steps 5 --warmup 6 --transport $tr --no-e2e >> gpurun_out/ab_$tr.json 2>> gpurun_out/ab_$tr.err
  echo "$tr exit $?" >> gpurun_out/ab.log
done
