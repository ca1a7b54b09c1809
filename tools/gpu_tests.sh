# run the GPU suite in chunks with per-chunk timeouts; logs in gpurun_out/
export PYTHONPATH=$PWD
for k in "$@"; do
  timeout 900 python -m pytest tests/ -q -m gpu -k "$k" -p no:cacheprovider -x > gpurun_out/t_$k.log 2>&1
  echo "$k exit $?" >> gpurun_out/summary.txt
done
