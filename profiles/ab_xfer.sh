# host-transfer A/B at c3 (1 GPU): threads vs hybrid (upload fraction f gathered by the GPU, tail scatter on)
for rep in 1 2 3 4; do
for v in threads:0:1 hybrid:0.2:1 hybrid:0.1:1; do
  IFS=: read x f sc <<< "$v"
  OMB_HOST_XFER=$x OMB_GATHER_FRAC=$f OMB_SCATTER_TAIL=$sc python bench.py --steps 2 --warmup 3 --efficiency-steps 0 \
    --e2e-steps 24 --no-cpu-baseline > gpurun_out/abx4_${x}_${f}_${sc}_$rep.json 2>/dev/null
done; done
