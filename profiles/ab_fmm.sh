#!/usr/bin/env bash
# A/B of the FMM target order on one box: c5g (self-gravitating star, 128^3), OMB_FMM_ORDER=0/1
TAG=$1
mkdir -p gpurun_out
for rep in 1 2; do
  for o in 0 1; do
    OMB_FMM_ORDER=$o python bench.py --config c5g --steps 5 --warmup 3 --e2e-steps -1 > gpurun_out/${TAG}_o${o}_$rep.json 2>/dev/null
  done
done
