#!/bin/bash
# one GPU: speculation parity tests and C5 time-to-plan with / without the same-device auxiliary context
mkdir -p gpurun_out
python -m pytest tests/test_engine_schedule.py -x -q > gpurun_out/spec_tests.log 2>&1; echo rc=$? >> gpurun_out/spec_tests.log
for r in 1 2; do
  GPLAN_SPECULATE=0 python tools/ttp_native.py c5_1024gpu/eta=2 | sed 's/^/off /'
  python tools/ttp_native.py c5_1024gpu/eta=2 | sed 's/^/on  /'
done > gpurun_out/spec_ab.log 2>&1
