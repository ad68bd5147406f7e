#!/bin/bash
# A/B of the train-batch lane policy on the C5 schedule (1 GPU): alternating runs
mkdir -p gpurun_out
python -m pytest tests/test_engine_schedule.py tests/test_engine_train.py -x -q > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
for r in 1 2; do
  GPLAN_BIG_LANE=0 python tools/ttp_native.py c5_1024gpu/eta=2 | sed 's/^/lanes-rr /'
  python tools/ttp_native.py c5_1024gpu/eta=2 | sed 's/^/big-lane /'
done > gpurun_out/ttp_ab.log 2>&1
GPLAN_PROFILE=1 python tools/ttp_native.py c5_1024gpu/eta=2 > gpurun_out/ttp_1dev_prof.log 2>&1
