set -x
for rep in 1 2; do
for v in threads hybrid:0.05 hybrid:0.1 hybrid:0.15 hybrid:0.2; do
  x=${v%%:*}; f=${v#*:}; [ "$f" = "$v" ] && f=0
  OMB_HOST_XFER=$x OMB_GATHER_FRAC=$f python bench.py --steps 5 --warmup 3 --efficiency-steps 0 --no-cpu-baseline > gpurun_out/abx_${x}_${f}_$rep.json 2>/dev/null
done; done
for c in c2; do for v in threads hybrid:0.1; do x=${v%%:*}; f=${v#*:}; [ "$f" = "$v" ] && f=0
  OMB_HOST_XFER=$x OMB_GATHER_FRAC=$f python bench.py --config c2 --steps 5 --warmup 3 --efficiency-steps 0 --no-cpu-baseline > gpurun_out/abx_${c}_${x}_${f}.json 2>/dev/null; done; done
