#!/bin/bash
# Round-end 1-GPU evidence: GPU suite (product and bounds-checked builds), smoke, bench line,
# reference arm, launch list of the bench command
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
GPLAN_LIB=$PWD/variants/libgplan_checks.so python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_checks.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_checks.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-units > gpurun_out/ncu.log 2>&1
