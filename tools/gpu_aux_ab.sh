#!/bin/bash
# A/B: speculative partitions on an auxiliary context on the SAME (single) GPU
mkdir -p gpurun_out
for r in 1 2; do
  python tools/ttp_native.py c5_1024gpu/eta=2 --devices 0 | sed 's/^/plain /'
  GPLAN_AUX_SAME_DEVICE=1 python tools/ttp_native.py c5_1024gpu/eta=2 --devices 0 | sed 's/^/aux   /'
done > gpurun_out/aux_ab.log 2>&1
GPLAN_AUX_SAME_DEVICE=1 python -m pytest tests/test_engine_schedule.py -x -q > gpurun_out/aux_tests.log 2>&1; echo rc=$? >> gpurun_out/aux_tests.log
