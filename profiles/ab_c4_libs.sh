#!/usr/bin/env bash
# A/B of library builds on c4 (AMR Sedov): bash profiles/ab_c4_libs.sh TAG lib1.so lib2.so ...
TAG=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in "$@"; do
    n=$(basename $lib .so)
    OMB_LIB_PATH=$lib python bench.py --config c4 --steps 30 --e2e-steps -1 --no-cpu-baseline > gpurun_out/${TAG}_${n}_$rep.json 2>/dev/null
  done
done
