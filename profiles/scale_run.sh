#!/usr/bin/env bash
# The bench contract's scaling commands on one box (run under gpurun --gpus N):
#   bash profiles/scale_run.sh TAG "1 2 4"
TAG=$1; NS=${2:-"1 2 4"}
mkdir -p gpurun_out
for n in $NS; do
  if [ "$n" = 1 ]; then
    python bench.py > gpurun_out/${TAG}_n1.json 2> gpurun_out/${TAG}_n1.err
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) \
      bench.py --gpus $n > gpurun_out/${TAG}_n$n.json 2> gpurun_out/${TAG}_n$n.err
  fi
done
