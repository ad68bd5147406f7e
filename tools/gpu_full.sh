timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash tools/variants.sh
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log | cut -c1-400
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttp > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_layout_scan -s 1 -c 1 -o gpurun_out/k1_final2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-ttp > gpurun_out/ncu_full.log 2>&1
ls gpurun_out | grep k1_final2
