#!/usr/bin/env bash
# A/B of environment switches on one box: bash profiles/ab_env.sh TAG "VAR=a" "VAR=b" ...
# (c2 and c3, 30 steps each, two rounds alternating)
TAG=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  for kv in "$@"; do
    n=$(echo "$kv" | tr '=,' '__')
    env $kv python bench.py --config c2 --steps 30 --e2e-steps -1 --no-cpu-baseline > gpurun_out/${TAG}_${n}_c2_$rep.json 2>/dev/null
    env $kv python bench.py --steps 30 --e2e-steps -1 --no-cpu-baseline > gpurun_out/${TAG}_${n}_c3_$rep.json 2>/dev/null
  done
done
