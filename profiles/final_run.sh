#!/usr/bin/env bash
# Round-end evidence on one box (run under gpurun --gpus 4): the GPU tests, the bench contract's
# commands at N = 1, 2, 4 (c3), the reference arm, and the other configs on one GPU.
TAG=${1:-r02final}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo pytest_rc=$? >> gpurun_out/${TAG}_pytest.log
bash profiles/scale_run.sh ${TAG} "1 2 4"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
for cfg in c2 c4 c5; do
  python bench.py --config $cfg --no-cpu-baseline > gpurun_out/${TAG}_$cfg.json 2> gpurun_out/${TAG}_$cfg.err
done
python bench.py --config c5g --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/${TAG}_c5g.json 2> gpurun_out/${TAG}_c5g.err
python bench.py --subgrid 16 --steps 30 --e2e-steps 2 --no-cpu-baseline > gpurun_out/${TAG}_n16.json 2> gpurun_out/${TAG}_n16.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --gpus 2 --config c4 > gpurun_out/${TAG}_c4_n2.json 2> gpurun_out/${TAG}_c4_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 \
  bench.py --gpus 2 --config c5g --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/${TAG}_c5g_n2.json 2> gpurun_out/${TAG}_c5g_n2.err
