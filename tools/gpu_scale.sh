# 2- and 4-GPU bench lines of the current build + C5 time-to-best-plan on 1 and 4 GPUs (one gpurun --gpus 4 call)
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2950$N bench.py --gpus $N --no-ttp > gpurun_out/bench_${N}gpu.log 2>&1; tail -1 gpurun_out/bench_${N}gpu.log | cut -c1-300
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29510 bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_ref4.log 2>&1; tail -1 gpurun_out/bench_ref4.log | cut -c1-300
timeout 600 python tools/ttp_native.py c5_1024gpu/eta=2 --devices 0,1,2,3 > gpurun_out/ttp4.log 2>&1; cat gpurun_out/ttp4.log | cut -c1-600
timeout 600 python tools/ttp_native.py c5_1024gpu/eta=2 > gpurun_out/ttp1.log 2>&1; cat gpurun_out/ttp1.log | cut -c1-600
