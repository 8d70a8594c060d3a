#!/usr/bin/env bash
# ncu evidence for the default workload (c3, 1 GPU): the launch list and one --set full capture of k_stage.
# Each ncu command runs after the same command exited 0 without ncu.
TAG=${1:-r02final}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps -1 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    $CMD > gpurun_out/${TAG}_ncu_list.log 2>&1
$CMD > gpurun_out/${TAG}_plain2.json 2> gpurun_out/${TAG}_plain2.err && \
ncu --set full --clock-control none --import-source on -k regex:k_stage -s 9 -c 1 -o gpurun_out/${TAG}_k_stage_c3 \
    $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
