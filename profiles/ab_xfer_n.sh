# host-transfer A/B at c3 on N GPUs of one box: mapped (GPU moves everything) vs hybrid fractions
N=${1:-4}
for rep in 1 2; do
for v in mapped:0 hybrid:0.5 hybrid:0.7; do
  IFS=: read x f <<< "$v"
  OMB_HOST_XFER=$x OMB_GATHER_FRAC=$f python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29600 + rep)) bench.py --gpus $N --steps 3 --warmup 3 \
    --efficiency-steps 0 --e2e-steps 12 > gpurun_out/abxn${N}_${x}_${f}_$rep.json 2>gpurun_out/abxn${N}_${x}_${f}_$rep.err
done; done
