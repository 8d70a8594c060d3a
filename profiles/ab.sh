#!/usr/bin/env bash
# A/B of library builds on the same box (gpurun, 1 GPU): bash profiles/ab.sh TAG lib1.so lib2.so ...
# (c3 30 steps + c2 30 steps per build, two rounds alternating); summarise with profiles/ab_summary.py TAG.
# Variant builds: python -c "from paper_2107_10987_b200 import build; build.build(force=True, out='exp/lib_X.so', defines=(...))"
TAG=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in "$@"; do
    n=$(basename $lib .so)
    OMB_LIB_PATH=$lib python bench.py --steps 30 --e2e-steps -1 --no-cpu-baseline > gpurun_out/${TAG}_${n}_c3_$rep.json 2>/dev/null
    OMB_LIB_PATH=$lib python bench.py --config c2 --steps 30 --e2e-steps -1 --no-cpu-baseline > gpurun_out/${TAG}_${n}_c2_$rep.json 2>/dev/null
  done
done
