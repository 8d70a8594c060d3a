for rep in 1 2 3; do for x in threads hybrid; do
OMB_HOST_XFER=$x python bench.py --config c4 --steps 5 --warmup 3 --e2e-steps 16 --no-cpu-baseline --efficiency-steps 0 > gpurun_out/c4x_${x}_$rep.json 2>/dev/null
done; done
