#!/bin/bash
# One GPU iteration: parity subset, bench, ncu capture of K1. Usage: tools/gpu_iter.sh TAG [pytest -k expr]
TAG=${1:-iter}; K=${2:-"golden or slices or ranges"}
timeout 400 python -m pytest tests -x -q -m gpu -k "$K" 2>&1 | tail -2
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-ttp > gpurun_out/bench_$TAG.log 2>&1
tail -1 gpurun_out/bench_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'k1_ms', d['roofline']['k1_ms_per_step'], 'k2_ms', d['roofline']['k2_ms_per_step'], 'frac', d['roofline']['frac'], 'winner', d['winner'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_layout_scan -s 1 -c 1 -o gpurun_out/k1_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-ttp > gpurun_out/ncu_$TAG.log 2>&1
ls gpurun_out | grep "k1_$TAG"
