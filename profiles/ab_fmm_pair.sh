#!/usr/bin/env bash
# A/B of the paired pass 0 (both stage solves in one pass over the lists) on c5g: OMB_FMM_PAIR=0/1
TAG=$1
mkdir -p gpurun_out
for rep in 1 2; do
  for v in 0 1; do
    OMB_FMM_PAIR=$v python bench.py --config c5g --steps 5 --warmup 3 --e2e-steps -1 > gpurun_out/${TAG}_pair${v}_$rep.json 2>/dev/null
  done
done
