#!/usr/bin/env bash
# A/B of library builds on c5g (self-gravitating star): bash profiles/ab_fmm_libs.sh TAG lib1.so lib2.so ...
TAG=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in "$@"; do
    n=$(basename $lib .so)
    OMB_LIB_PATH=$lib python bench.py --config c5g --steps 5 --warmup 3 --e2e-steps -1 > gpurun_out/${TAG}_${n}_$rep.json 2>/dev/null
  done
done
