#!/usr/bin/env bash
# One ncu --set full capture of one k_stage launch at config c2 (run under gpurun, 1 GPU):
#   bash profiles/ncu_stage.sh TAG
# The same command runs once without ncu first (it must exit 0), then under ncu.
set -euo pipefail
TAG=${1:-r02}
mkdir -p gpurun_out
CMD="python bench.py --config c2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err
ncu --set full --clock-control none --import-source on -k regex:k_stage -s 9 -c 1 \
    -o gpurun_out/${TAG}_k_stage $CMD > gpurun_out/${TAG}_ncu.log 2>&1
