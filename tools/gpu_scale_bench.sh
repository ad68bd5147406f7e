#!/bin/bash
# 2- and 4-GPU bench lines (torchrun, one rank per GPU); the 4-GPU line includes the
# time-to-best-plan leg on a 4-device context. Run under gpurun --gpus 4.
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29504 \
  bench.py --gpus 4 > gpurun_out/bench_4gpu.json 2> gpurun_out/bench_4gpu.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29502 \
  bench.py --gpus 2 --no-ttp > gpurun_out/bench_2gpu.json 2> gpurun_out/bench_2gpu.err
